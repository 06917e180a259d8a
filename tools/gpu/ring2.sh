set -u
timeout 600 python tools/perf.py C5 C5:4000000 --reps 2 --out gpurun_out/ring2.json > gpurun_out/ring2.log 2>&1; echo "rc=$?" >> gpurun_out/ring2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C5 or scaled or determinism" > gpurun_out/ring2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ring2_tests.log
