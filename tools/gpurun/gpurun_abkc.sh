#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for lib in ab/libfsil_base.so paper_2303_14102_b200/libfsil.so; do
  for c in "C2 1000000" "C1 100000"; do
    FSIL_LIB_PATH=$PWD/$lib timeout 200 python tools/gpurun/gpurun_ab.py $c 2>&1 | tail -1
  done
done
done
