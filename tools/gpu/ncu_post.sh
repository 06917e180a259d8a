set -u
python tools/perf.py C5:8000000 --reps 1 --out gpurun_out/np.json > gpurun_out/np_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"agg_piece_ring|exact_kernel|refine_tiled" -c 3 \
    -o gpurun_out/r02_post_c5_8m python tools/perf.py C5:8000000 --reps 1 --out gpurun_out/np.json > gpurun_out/ncu_np.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_np.log
