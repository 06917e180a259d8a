set -u
timeout 300 python tools/perf.py C5:8000000 --reps 1 --out gpurun_out/l8.json > gpurun_out/l8_plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l8_launches.csv \
    python tools/perf.py C5:8000000 --reps 1 --out gpurun_out/l8n.json > gpurun_out/l8_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/l8_ncu.log
