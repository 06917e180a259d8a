#!/bin/bash
# Source-level ncu captures (inst_executed per line) of the two C2 kernels.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:score_tc -s 1 -c 1 -o gpurun_out/src_c2_score_tc \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_src1.log 2>&1; echo "score rc=$?"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:agg_stage -s 1 -c 1 -o gpurun_out/src_c2_agg \
  python tools/gpurun/gpurun_prof.py C2 1000000 2 > gpurun_out/ncu_src2.log 2>&1; echo "agg rc=$?"
