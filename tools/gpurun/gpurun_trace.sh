#!/bin/bash
cd "$GRAFT_REPO_ROOT"
FSIL_TC_TRACE=1 FSIL_LIB_PATH=$PWD/ab/libfsil_trace.so timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | grep -A 56 "tc trace" | tail -30
