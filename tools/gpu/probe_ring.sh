set -u
./tools/mma_rate > gpurun_out/mma_rate.log 2>&1; echo "rc=$?" >> gpurun_out/mma_rate.log
python tools/perf.py C5:4000000 --reps 1 --out gpurun_out/pr.json > gpurun_out/pr_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"agg_piece_ring|label_scatter|label_count|exact_kernel" -s 8 -c 4 \
    -o gpurun_out/r02_agg_c5_4m python tools/perf.py C5:4000000 --reps 1 --out gpurun_out/pr.json > gpurun_out/ncu_ring.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_ring.log
