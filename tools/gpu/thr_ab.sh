set -u
timeout 600 python tools/thr_check.py > gpurun_out/thr_check.log 2>&1; echo "rc=$?" >> gpurun_out/thr_check.log
timeout 600 python tools/perf.py C4:20000000 C4 --reps 3 --out gpurun_out/perf_thr.json > gpurun_out/perf_thr.log 2>&1; echo "rc=$?" >> gpurun_out/perf_thr.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4_20m.csv python tools/perf.py C4:20000000 --reps 1 --out gpurun_out/perf_ncu.json > gpurun_out/ncu_c4.log 2>&1
python - <<'PY' > gpurun_out/launches_c4_20m.txt 2>&1
import csv
rows = [r for r in csv.reader(open('gpurun_out/launches_c4_20m.csv')) if len(r) > 10]
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
names = [(r[ki][:70], float(r[vi].replace(',', ''))) for r in rows[1:]]
for n, v in names[-19:]: print(f"{v/1e3:10.1f} us  {n}")
PY
