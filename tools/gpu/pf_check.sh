set -u
for spec in C5,600 C5,3000 C5,20000 2000,768,300,cosine 3000,512,1000,sqeuclid 1000,256,700,cosine 517,320,513,sqeuclid; do
  timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/pf_dbg.log 2>&1; echo "$spec rc=$?" >> gpurun_out/pf_dbg.log
done
FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/pf_prof.json 2>&1 | grep profile | tail -1 >> gpurun_out/pf_dbg.log
timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/pf_perf.json > gpurun_out/pf_perf.log 2>&1; echo "rc=$?" >> gpurun_out/pf_perf.log
FSIL_TC_PAIR_PF=0 timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/pf_perf0.json > gpurun_out/pf_perf0.log 2>&1
