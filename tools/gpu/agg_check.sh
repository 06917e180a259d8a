set -u
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "scaled or full_size or determinism or batched or validation or shard" > gpurun_out/agg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/agg_tests.log
timeout 900 python tools/perf.py C3 C4 C5 --reps 3 --out gpurun_out/perf_agg.json > gpurun_out/perf_agg.log 2>&1; echo "rc=$?" >> gpurun_out/perf_agg.log
FSIL_AGG_CUB=1 FSIL_AGG_RING=0 timeout 900 python tools/perf.py C3 C4 C5 --reps 3 --out gpurun_out/perf_agg_old.json > gpurun_out/perf_agg_old.log 2>&1; echo "rc=$?" >> gpurun_out/perf_agg_old.log
python tools/perf.py C5:151552 --reps 1 --out gpurun_out/perf_c5s.json > gpurun_out/plain_c5s.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"score_tc_pair|agg_piece_ring|label_" -s 6 -c 6 \
    -o gpurun_out/r02_pair_c5s python tools/perf.py C5:151552 --reps 1 --out gpurun_out/perf_c5s.json > gpurun_out/ncu_c5s.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_c5s.log
