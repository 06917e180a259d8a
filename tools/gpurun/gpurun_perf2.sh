#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python tools/gpurun/gpurun_perf.py > gpurun_out/perf.log 2>&1; echo "perf rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
