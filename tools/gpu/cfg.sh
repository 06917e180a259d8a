set -u
for cfg in "3 2 2" "2 3 2" "3 3 1" "2 2 3"; do
  set -- $cfg
  FSIL_TC_PAIR_NS=$1 FSIL_TC_PAIR_NB=$2 FSIL_TC_PAIR_NX=$3 FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/cfg.json 2>&1 | grep profile | tail -1 | cut -c1-260 >> gpurun_out/cfg.log
  echo "$cfg $(FSIL_TC_PAIR_NS=$1 FSIL_TC_PAIR_NB=$2 FSIL_TC_PAIR_NX=$3 timeout 300 python tools/perf.py C5:8000000 --reps 2 --out gpurun_out/cfg8.json 2>&1 | tail -1 | grep -o '"ms_score_kernel": [0-9.]*')" >> gpurun_out/cfg.log
done
