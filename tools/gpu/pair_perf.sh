set -u
timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/perf_pair.json > gpurun_out/perf_pair.log 2>&1; echo "rc=$?" >> gpurun_out/perf_pair.log
FSIL_TC_PAIR=0 timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/perf_nopair.json > gpurun_out/perf_nopair.log 2>&1; echo "rc=$?" >> gpurun_out/perf_nopair.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C5 or streaming or scaled or near_ties or mixed_norms" > gpurun_out/pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair_tests.log
