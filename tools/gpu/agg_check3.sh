set -u
timeout 900 python tools/perf.py C3 C4 C5 --reps 3 --out gpurun_out/perf_agg4.json > gpurun_out/perf_agg4.log 2>&1; echo "rc=$?" >> gpurun_out/perf_agg4.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "scaled or determinism or strong_scaling or k_speculation or validation" > gpurun_out/agg4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/agg4_tests.log
