set -u
for e in 0 1 2; do
  echo "EXP=$e $(FSIL_TC_EXP=$e timeout 300 python tools/perf.py C4:20000000 --reps 3 --out gpurun_out/ab.json 2>&1 | tail -1 | grep -o '"ms": [0-9.]*\|"ms_score_kernel": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/exp.log
done
