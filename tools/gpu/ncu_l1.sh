set -u
python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/nl1.json > gpurun_out/nl1_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"score_tc_pair" -s 2 -c 1 \
    -o gpurun_out/r02_pair_l1d_c5_1m python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/nl1.json > gpurun_out/ncu_nl1.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_nl1.log
