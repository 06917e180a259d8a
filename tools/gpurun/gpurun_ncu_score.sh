#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:score_tc -s 1 -c 1 -o gpurun_out/r01_c2_score_tc \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_c2s.log 2>&1; echo "c2 score rc=$?"
