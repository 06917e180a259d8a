#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do for lib in paper_2303_14102_b200/libfsil.so ab/libfsil_br8.so; do FSIL_LIB_PATH=$PWD/$lib timeout 300 python tools/gpurun/gpurun_phases.py C2 2>&1 | sed "s|^|$(basename $lib) |" | cut -c1-220; done; done
