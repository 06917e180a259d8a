#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for ns in 2 3 4 5; do FSIL_TC_NSTG=$ns timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -1 | sed "s/^/nstg=$ns /"; done
