# ncu --set full of the tcgen05 scoring kernel at C5 (8 tiles per SM) and C4 (211 tiles per SM);
# each command first exits 0 without ncu.
set -u
for c in C5:151552 C4:4000000; do
  tag=$(echo $c | tr ':' '_')
  python tools/perf.py $c --reps 1 --out gpurun_out/perf_$tag.json > gpurun_out/plain_$tag.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:score_tc -s 2 -c 1 \
      -o gpurun_out/r02_score_$tag python tools/perf.py $c --reps 1 --out gpurun_out/perf_$tag.json \
      > gpurun_out/ncu_$tag.log 2>&1
  echo "$c rc=$?" >> gpurun_out/ncu_$tag.log
done
