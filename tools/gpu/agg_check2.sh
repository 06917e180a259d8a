set -u
timeout 900 python tools/perf.py C3 C4 C5 --reps 3 --out gpurun_out/perf_agg2.json > gpurun_out/perf_agg2.log 2>&1; echo "rc=$?" >> gpurun_out/perf_agg2.log
FSIL_EXACT_SORTED=0 timeout 600 python tools/perf.py C5 --reps 2 --out gpurun_out/perf_agg2_nosort.json > gpurun_out/perf_agg2_nosort.log 2>&1; echo "rc=$?" >> gpurun_out/perf_agg2_nosort.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/agg2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/agg2_tests.log
