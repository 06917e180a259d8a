set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "threshold or adversarial" > gpurun_out/ws_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ws_tests.log
for w in 0 4 8 0 4; do
  echo "WSHIFT=$w $(FSIL_TC_WSHIFT=$w timeout 300 python tools/perf.py C4:20000000 --reps 5 --out gpurun_out/ab.json 2>&1 | tail -1 | grep -o '"ms": [0-9.]*\|"ms_score_kernel": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/ws.log
done
