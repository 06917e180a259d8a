set -u
for spec in C5,600 C5,3000 C5,20000 2000,768,300,cosine 3000,512,1000,sqeuclid 1000,256,700,cosine 517,320,513,sqeuclid; do
  timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/l1_dbg.log 2>&1; echo "$spec rc=$?" >> gpurun_out/l1_dbg.log
done
FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/l1_prof.json 2>&1 | grep profile | tail -1 >> gpurun_out/l1_dbg.log
timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/l1_perf.json > gpurun_out/l1_perf.log 2>&1; echo "rc=$?" >> gpurun_out/l1_perf.log
FSIL_TC_L1=2 timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/l1_perf2.json > gpurun_out/l1_perf2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/l1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l1_tests.log
