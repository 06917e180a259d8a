set -u
for cfg in "3 3" "4 2"; do
  set -- $cfg
  FSIL_TC_PAIR_NS=$1 FSIL_TC_PAIR_NB=$2 FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/ls.json 2>&1 | grep profile | tail -1 >> gpurun_out/l1_stage.log
  FSIL_TC_PAIR_NS=$1 FSIL_TC_PAIR_NB=$2 timeout 300 python tools/perf.py C5:8000000 --reps 2 --out gpurun_out/ls_$1$2.json 2>&1 | tail -1 | cut -c1-300 >> gpurun_out/l1_stage.log
done
