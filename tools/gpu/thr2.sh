set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "threshold or adversarial" > gpurun_out/thr2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/thr2_tests.log
timeout 600 python tools/perf.py C4:20000000 --reps 10 --out gpurun_out/perf_thr2.json > gpurun_out/perf_thr2.log 2>&1; echo "rc=$?" >> gpurun_out/perf_thr2.log
