#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for c in "C5 200000" "C4 2000000" "C3 2000000"; do
  for r in 0 1; do FSIL_TC_RING=$r timeout 300 python tools/gpurun/gpurun_ab.py $c 2>&1 | tail -1 | sed "s/^/ring=$r /"; done
done
