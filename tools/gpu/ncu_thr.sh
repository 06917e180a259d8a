set -u
c=C4:4000000
python tools/perf.py $c --reps 1 --out gpurun_out/perf_c4_4m.json > gpurun_out/plain_c4_4m.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:score_tc -s 2 -c 1 \
    -o gpurun_out/r02_C4_thr_score python tools/perf.py $c --reps 1 --out gpurun_out/perf_c4_4m.json \
    > gpurun_out/ncu_c4_thr.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c4_thr.log
ncu --set full --clock-control none --import-source on -k regex:thr_kernel -s 2 -c 1 \
    -o gpurun_out/r02_C4_thr_kernel python tools/perf.py $c --reps 1 --out gpurun_out/perf_c4_4m.json \
    > gpurun_out/ncu_c4_thrk.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c4_thrk.log
