#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for lib in ab/libfsil_prev.so ab/libfsil_r40.so ab/libfsil_r48.so paper_2303_14102_b200/libfsil.so; do
  FSIL_LIB_PATH=$PWD/$lib timeout 200 python tools/gpurun/gpurun_ab.py C4 2000000 2>&1 | tail -1
  FSIL_LIB_PATH=$PWD/$lib timeout 200 python tools/gpurun/gpurun_ab.py C3 2000000 2>&1 | tail -1
done
