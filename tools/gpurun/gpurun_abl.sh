#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for lib in paper_2303_14102_b200/libfsil.so ab/libfsil_aall.so ab/libfsil_aconv.so ab/libfsil_ascanfin.so; do
  FSIL_LIB_PATH=$PWD/$lib timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -1
done
