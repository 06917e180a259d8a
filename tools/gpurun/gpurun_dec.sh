#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for d in 0 1; do FSIL_TC_DECOUPLE=$d timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -1 | sed "s/^/dec=$d /"; done
timeout 300 python tools/gpurun/gpurun_phases.py C1 C2 C2 C3:2000000 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
