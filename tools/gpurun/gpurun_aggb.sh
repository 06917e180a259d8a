#!/bin/bash
# A/B of the two-phase batched aggregation (FSIL_AGG_BATCH=1, default) against agg_stage.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in 0 1; do FSIL_AGG_BATCH=$v timeout 300 python tools/gpurun/gpurun_phases.py C1 C2 C2 2>&1 | sed "s/^/batch=$v /"; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:agg_batch -s 1 -c 1 -o gpurun_out/src_c2_aggb2 \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_aggb.log 2>&1; echo "aggb rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
