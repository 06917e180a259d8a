set -u
FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/diag1.json 2>&1 | grep profile | tail -1 >> gpurun_out/diag.log
FSIL_TC_PROFILE=2 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/diag2.json 2>&1 | grep -E "profile|Error|error" | tail -3 >> gpurun_out/diag.log
