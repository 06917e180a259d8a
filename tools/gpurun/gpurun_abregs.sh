#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for lib in paper_2303_14102_b200/libfsil.so ab/libfsil_e128.so ab/libfsil_e136.so; do
  for c in "C2 1000000" "C3 2000000" "C4 4000000"; do
    FSIL_LIB_PATH=$PWD/$lib timeout 200 python tools/gpurun/gpurun_ab.py $c 2>&1 | tail -1
  done
done
done
