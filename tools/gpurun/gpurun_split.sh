#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for sp in 0 1; do FSIL_TC_SPLIT=$sp timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -1 | sed "s/^/split=$sp /"; done
for sp in 0 1; do FSIL_TC_SPLIT=$sp FSIL_LIB_PATH=$PWD/ab/libfsil_aall.so timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -1 | sed "s/^/aall split=$sp /"; done
