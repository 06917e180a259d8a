#!/bin/bash
# Full GPU suite + per-phase timings of C1/C2 (and C3 at 2M rows).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python tools/gpurun/gpurun_phases.py C1 C2 C2 C3:2000000 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
