set -u
for cfg in "4 2" "3 3" "3 2"; do
  set -- $cfg
  FSIL_TC_PAIR_NS=$1 FSIL_TC_PAIR_NB=$2 FSIL_TC_PROFILE=1 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/st.json 2>&1 | grep profile | tail -1 >> gpurun_out/pair_stages.log
  FSIL_TC_PAIR_NS=$1 FSIL_TC_PAIR_NB=$2 python tools/perf.py C5:4000000 --reps 3 --out gpurun_out/st_$1$2.json 2>&1 | tail -1 | cut -c1-400 >> gpurun_out/pair_stages.log
done
python tools/perf.py C3 C4 --reps 3 --out gpurun_out/perf_agg3.json > gpurun_out/perf_agg3.log 2>&1
