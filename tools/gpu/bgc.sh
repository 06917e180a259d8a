set -u
for spec in C5,3000 C5,20000 2000,768,300,cosine 3000,512,1000,sqeuclid 517,320,513,sqeuclid 9000,320,2100,cosine 30000,136,513,sqeuclid 5000,100,700,cosine; do
  timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/bgc.log 2>&1
done
FSIL_TC_L1=2 timeout 120 python tools/dbg_shapes.py C5,20000 >> gpurun_out/bgc.log 2>&1
FSIL_TC_L1=3 timeout 120 python tools/dbg_shapes.py C5,20000 >> gpurun_out/bgc.log 2>&1
FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/bgc_prof.json 2>&1 | grep profile | tail -1 >> gpurun_out/bgc.log
timeout 300 python tools/perf.py C5:8000000 --reps 2 --out gpurun_out/bgc8.json 2>&1 | tail -1 | cut -c1-400 >> gpurun_out/bgc.log
