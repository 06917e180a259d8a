#!/bin/bash
# Round evidence: bench line, reference arm, bench launch list, ncu captures of the top kernels.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:score_tc -s 1 -c 1 -o gpurun_out/r01_c2_score_tc \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_c2s.log 2>&1; echo "c2 score rc=$?"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:agg_batch -s 1 -c 1 -o gpurun_out/r01_c2_agg_batch \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_c2a.log 2>&1; echo "c2 agg rc=$?"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:score_ffma -s 1 -c 1 -o gpurun_out/r01_c2_score_ffma \
  python tools/gpurun/gpurun_prof.py C2 1000000 1 > gpurun_out/ncu_c2f.log 2>&1; echo "c2 ffma rc=$?"
for c in "C3 2000000" "C4 2000000" "C5 200000"; do
  set -- $c
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:score_tc -s 1 -c 1 -o gpurun_out/r01_${1}_score_tc \
    python tools/gpurun/gpurun_prof.py $1 $2 2 > gpurun_out/ncu_$1.log 2>&1; echo "$1 rc=$?"
done
timeout 1200 python tools/gpurun/gpurun_perf.py > gpurun_out/perf.log 2>&1; echo "perf rc=$?"
