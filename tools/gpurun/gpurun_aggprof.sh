#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:agg_batch -s 1 -c 1 -o gpurun_out/src_c2_aggb \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_aggb.log 2>&1; echo "aggb rc=$?"
