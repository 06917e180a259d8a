set -u
timeout 600 python tools/thr_check.py > gpurun_out/thr_check.log 2>&1; echo "rc=$?" >> gpurun_out/thr_check.log
for cfg in "2 4 1" "2 4 3" "1 4 1"; do
  set -- $cfg
  echo "NB=$1 NS=$2 L1=$3 $(FSIL_THR_NB=$1 FSIL_THR_NS=$2 FSIL_THR_L1=$3 timeout 300 python tools/perf.py C4:20000000 --reps 3 --out gpurun_out/ab.json 2>&1 | tail -1 | grep -o '"ms": [0-9.]*\|"flagged_rows": [0-9]*\|"ms_score": [0-9.]*\|"ms_refine": [0-9.]*\|"ms_score_kernel": [0-9.]*\|"pair_rows": [0-9]*' | tr '\n' ' ')" >> gpurun_out/thr_ab.log
done
FSIL_TC_PROFILE=1 timeout 300 python tools/perf.py C4:20000000 --reps 1 --out gpurun_out/perf_thr_prof.json 2>&1 | grep -i "profile" | tail -1 >> gpurun_out/thr_ab.log
