#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"densify" -s 0 -c 6 -o gpurun_out/small \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_small.log 2>&1; echo "rc=$?"
