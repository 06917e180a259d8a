#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2 3; do for lib in ab/libfsil_prev.so paper_2303_14102_b200/libfsil.so; do FSIL_LIB_PATH=$PWD/$lib timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -1; done; done
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "batched or determinism or c2" 2>&1 | tail -2
