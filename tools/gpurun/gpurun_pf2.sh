#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for lib in ab/libfsil_prev.so paper_2303_14102_b200/libfsil.so; do
  FSIL_LIB_PATH=$PWD/$lib timeout 300 python tools/gpurun/gpurun_phases.py C2 2>&1 | sed "s|^|$lib |"
done; done
FSIL_TC_TRACE=1 FSIL_LIB_PATH=$PWD/ab/libfsil_trace.so timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | grep -A 56 "tc trace" | tail -8
