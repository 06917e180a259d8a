#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do for v in 0 1; do FSIL_AGG_REG=$v timeout 300 python tools/gpurun/gpurun_phases.py C2 C1 2>&1 | sed "s/^/reg=$v /"; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
