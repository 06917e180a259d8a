set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not full_size" > gpurun_out/dens_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dens_tests.log
timeout 600 python tools/perf.py C1 C2 C3 C4:20000000 C5:4000000 --reps 10 --out gpurun_out/perf_dens.json > gpurun_out/perf_dens.log 2>&1; echo "rc=$?" >> gpurun_out/perf_dens.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c4d.csv python tools/perf.py C4:20000000 --reps 1 --out gpurun_out/perf_ncu.json > gpurun_out/ncu_c4d.log 2>&1
python - <<'PY' > gpurun_out/launches_c4d.txt 2>&1
import csv
rows = [r for r in csv.reader(open('gpurun_out/launches_c4d.csv')) if len(r) > 10]
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
names = [(r[ki][:70], float(r[vi].replace(',', ''))) for r in rows[1:]]
for n, v in names[-19:]: print(f"{v/1e3:10.1f} us  {n}")
PY
