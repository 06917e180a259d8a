# Per-config timing table (builder tool) plus the C2 / C1 launch lists
set -u
timeout 900 python tools/perf.py C1 C2 C3 C4 --reps 10 --out gpurun_out/perf_all.json > gpurun_out/perf_all.log 2>&1; echo "rc=$?" >> gpurun_out/perf_all.log
for cfg in C1 C2 C3; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$cfg.csv python tools/perf.py $cfg --reps 1 --out gpurun_out/perf_ncu.json > gpurun_out/ncu_$cfg.log 2>&1
python - $cfg <<'PY' > gpurun_out/launches_$cfg.txt 2>&1
import csv, sys
cfg = sys.argv[1]
rows = [r for r in csv.reader(open(f'gpurun_out/launches_{cfg}.csv')) if len(r) > 10]
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
names = [(r[ki][:90], float(r[vi].replace(',', ''))) for r in rows[1:]]
# the last call's launches: back to the last densify_collect
last = max(i for i, (n, v) in enumerate(names) if 'densify_collect' in n or 'densify_small' in n or 'densify' in n and 'collect' in n)
for n, v in names[last:]: print(f"{v/1e3:10.1f} us  {n}")
print(f"{sum(v for n, v in names[last:])/1e3:10.1f} us  total")
PY
done
