# Round-end evidence in one call: GPU tests, smoke, bench (both arms), launch list of the bench
# command, ncu --set full of the dominant kernels, per-config table.
set -u
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_ref.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python tools/perf.py C1 C2 C3 C4 --reps 10 --out gpurun_out/perf_all.json > gpurun_out/perf_all.log 2>&1; echo "rc=$?" >> gpurun_out/perf_all.log
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_short.log 2>&1 &&
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_C5.csv \
    python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
for c in C5:2000000 C4:4000000; do
  tag=$(echo $c | tr ':' '_')
  timeout 600 python tools/perf.py $c --reps 1 --out gpurun_out/perf_$tag.json > gpurun_out/plain_$tag.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_tc" -s 2 -c 1 \
      -o gpurun_out/r02f_score_$tag python tools/perf.py $c --reps 1 --out gpurun_out/perf_$tag.json \
      > gpurun_out/ncu_$tag.log 2>&1
  echo "$c rc=$?" >> gpurun_out/ncu_$tag.log
done
