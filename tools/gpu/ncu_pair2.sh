set -u
python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/np2.json > gpurun_out/np2_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"score_tc_pair" -s 2 -c 1 \
    -o gpurun_out/r02_pair_c5_1m python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/np2.json > gpurun_out/ncu_np2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_np2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pair_kernel_shapes or streaming" > gpurun_out/pair_shape_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair_shape_tests.log
