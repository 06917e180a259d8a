#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
FSIL_TC_PROFILE=1 timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -3
timeout 300 ncu --set full --import-source on --clock-control none -k regex:score_tc -s 1 -c 1 -o gpurun_out/src_c2_score_tc3 \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_src3.log 2>&1; echo "score rc=$?"
