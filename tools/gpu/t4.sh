timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "threshold" > gpurun_out/t4_tests.log 2>&1; echo rc=$? >> gpurun_out/t4_tests.log
timeout 300 python tools/perf.py C4:20000000 C4 --reps 5 --out gpurun_out/ab.json > gpurun_out/t4.log 2>&1
