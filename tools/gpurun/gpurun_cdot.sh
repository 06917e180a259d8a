#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python tools/gpurun/gpurun_phases.py C2 C2 C3:2000000 C4:2000000 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
