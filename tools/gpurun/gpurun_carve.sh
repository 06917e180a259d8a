#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for v in 0 1; do FSIL_CARVEOUT=$v timeout 300 python tools/gpurun/gpurun_phases.py C2 C2 2>&1 | sed "s/^/carve=$v /"; done
