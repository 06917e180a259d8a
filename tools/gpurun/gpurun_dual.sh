#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for d in 0 1; do FSIL_TC_DUAL=$d timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -1 | sed "s/^/dual=$d /"; done
for d in 0 1; do FSIL_TC_DUAL=$d timeout 200 python tools/gpurun/gpurun_ab.py C3 2000000 2>&1 | tail -1 | sed "s/^/dual=$d /"; done
FSIL_TC_TRACE=1 FSIL_LIB_PATH=$PWD/ab/libfsil_trace.so timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | grep -A 40 "tc trace" | head -40
