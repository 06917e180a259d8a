set -u
FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/lp.json 2>&1 | grep profile | tail -1 > gpurun_out/l1_prof2.log
FSIL_TC_L1=3 FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/lp.json 2>&1 | grep profile | tail -1 >> gpurun_out/l1_prof2.log
