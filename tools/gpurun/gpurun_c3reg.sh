#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for c in "C3 2000000" "C4 2000000" "C2 1000000"; do
  FSIL_LIB_PATH=$PWD/ab/libfsil_prev.so timeout 200 python tools/gpurun/gpurun_ab.py $c 2>&1 | tail -1
  for d in 0 1; do FSIL_TC_DUAL=$d timeout 200 python tools/gpurun/gpurun_ab.py $c 2>&1 | tail -1 | sed "s/^/dual=$d /"; done
done
