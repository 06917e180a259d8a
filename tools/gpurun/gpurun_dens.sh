#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
FSIL_LIB_PATH=$PWD/ab/libfsil_prev.so timeout 300 python tools/gpurun/gpurun_phases.py C2 2>&1 | sed "s/^/prev /"
timeout 300 python tools/gpurun/gpurun_phases.py C2 2>&1 | sed "s/^/map4 /"
FSIL_LIB_PATH=$PWD/ab/libfsil_cu8.so timeout 300 python tools/gpurun/gpurun_phases.py C2 2>&1 | sed "s/^/map4+cu8 /"
done
