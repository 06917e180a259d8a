set -u
FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/diag31.json 2>&1 | grep profile | tail -1 >> gpurun_out/diag3.log
FSIL_TC_PROFILE=2 timeout 300 python tools/perf.py C5:1000000 --reps 1 --out gpurun_out/diag32.json 2>&1 | grep -E "profile|Error|error" | tail -3 >> gpurun_out/diag3.log
timeout 300 python tools/perf.py C5:8000000 --reps 2 --out gpurun_out/d3_8.json 2>&1 | tail -1 | cut -c1-400 >> gpurun_out/diag3.log; for spec in C5,3000 C5,20000 2000,768,300,cosine 9000,320,2100,cosine; do timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/diag3.log 2>&1; done
