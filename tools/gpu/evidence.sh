set -u
timeout 900 python tools/cpu_table.py --out gpurun_out/cpu_table.json > gpurun_out/cpu_table.log 2>&1; echo "rc=$?" >> gpurun_out/cpu_table.log
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_short.log 2>&1 &&
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_C5.csv \
    python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
