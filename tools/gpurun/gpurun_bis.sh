#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for c in "C4 2000000" "C3 2000000" "C2 1000000"; do
for lib in ab/libfsil_prev.so paper_2303_14102_b200/libfsil.so; do
  FSIL_LIB_PATH=$PWD/$lib timeout 200 python tools/gpurun/gpurun_ab.py $c 2>&1 | tail -1
done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
