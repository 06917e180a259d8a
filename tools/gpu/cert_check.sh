set -u
for spec in C5,3000 C5,20000 2000,768,300,cosine 3000,512,1000,sqeuclid 1000,256,700,cosine; do
  timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/cert_dbg.log 2>&1; echo "$spec rc=$?" >> gpurun_out/cert_dbg.log
done
timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/cert_perf.json > gpurun_out/cert_perf.log 2>&1; echo "rc=$?" >> gpurun_out/cert_perf.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/cert_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cert_tests.log
