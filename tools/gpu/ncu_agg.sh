set -u
python tools/perf.py C5:8000000 --reps 1 --out gpurun_out/np.json > gpurun_out/np_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"agg_piece_ring" -c 1 \
    -o gpurun_out/r02_agg2_c5_8m python tools/perf.py C5:8000000 --reps 1 --out gpurun_out/np.json > gpurun_out/ncu_np.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_np.log
