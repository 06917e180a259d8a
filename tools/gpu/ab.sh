# A/B of prebuilt library variants under abl/ on one box: perf.py per variant, twice, interleaved
set -u
spec=${1:-C5:8000000}
cp paper_2303_14102_b200/libfsil.so abl/current.so
for rep in 1 2; do
  for v in abl/*.so; do
    [ "$v" = abl/current.so ] && continue
    cp $v paper_2303_14102_b200/libfsil.so
    echo "$v $(timeout 300 python tools/perf.py $spec --reps 2 --out gpurun_out/ab.json 2>&1 | tail -1 | cut -c1-330)" >> gpurun_out/ab.log
  done
done
cp abl/current.so paper_2303_14102_b200/libfsil.so
