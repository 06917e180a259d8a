set -u
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_8m.csv python tools/perf.py C5:8000000 --reps 1 --out gpurun_out/perf_ncu.json > gpurun_out/ncu_c5_8m.log 2>&1
python - <<'PY' > gpurun_out/launches_c5_8m.txt 2>&1
import csv
rows = [r for r in csv.reader(open('gpurun_out/launches_c5_8m.csv')) if len(r) > 10]
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
names = [(r[ki][:70], float(r[vi].replace(',', ''))) for r in rows[1:]]
last = max(i for i, (n, v) in enumerate(names) if 'densify_collect' in n)
for n, v in names[last:]: print(f"{v/1e3:10.1f} us  {n}")
PY
