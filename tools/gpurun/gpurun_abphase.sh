#!/bin/bash
# A/B per-phase timings: HEAD build (ab/libfsil_prev.so) against the working tree.
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for lib in ab/libfsil_prev.so paper_2303_14102_b200/libfsil.so; do
  echo "== $lib"; FSIL_LIB_PATH=$PWD/$lib timeout 300 python tools/gpurun/gpurun_phases.py C2 C2 C3:2000000 C4:4000000 2>&1 | tail -4
done
done
