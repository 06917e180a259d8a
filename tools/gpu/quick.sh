set -u
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python tools/perf.py C4:20000000 C4 --reps 5 --out gpurun_out/perf_quick.json > gpurun_out/perf_quick.log 2>&1; echo "rc=$?" >> gpurun_out/perf_quick.log
