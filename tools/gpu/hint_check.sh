set -u
for spec in C5,3000 C5,20000 2000,768,300,cosine 3000,512,1000,sqeuclid; do
  timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/hint_dbg.log 2>&1; echo "$spec rc=$?" >> gpurun_out/hint_dbg.log
done
FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/hint_prof.json 2>&1 | grep profile | tail -1 >> gpurun_out/hint_dbg.log
timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/hint_perf.json > gpurun_out/hint_perf.log 2>&1; echo "rc=$?" >> gpurun_out/hint_perf.log
