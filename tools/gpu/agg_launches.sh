set -u
for c in C3:2000000 C4:8000000; do
  tag=$(echo $c | tr ':' '_')
  python tools/perf.py $c --reps 1 --out gpurun_out/pl_$tag.json > gpurun_out/pl_$tag.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
      python tools/perf.py $c --reps 1 --out gpurun_out/pl_$tag.json > /dev/null 2>&1
  FSIL_AGG_CUB=1 python tools/perf.py $c --reps 1 --out gpurun_out/pl_cub_$tag.json > gpurun_out/pl_cub_$tag.log 2>&1 &&
  FSIL_AGG_CUB=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cub_$tag.csv \
      python tools/perf.py $c --reps 1 --out gpurun_out/pl_cub_$tag.json > /dev/null 2>&1
done
FSIL_TC_PROFILE=1 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/prof_c5.json > gpurun_out/prof_c5.log 2>&1
