#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for lib in ab/libfsil_prev.so paper_2303_14102_b200/libfsil.so; do
  FSIL_LIB_PATH=$PWD/$lib timeout 300 python tools/gpurun/gpurun_phases.py C3:10000000 C4:10000000 2>&1 | sed "s|^|$(basename $lib) |" | cut -c1-200
done; done
