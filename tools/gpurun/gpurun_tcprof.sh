#!/bin/bash
# Per-role wait profile of the tcgen05 scoring kernel (FSIL_TC_PROFILE) on scaled configs.
export FSIL_TC_PROFILE=1
for cfg in "C2 1000000" "C3 2000000" "C4 2000000" "C5 200000"; do
  timeout 120 python tools/gpurun/gpurun_prof.py $cfg 2 2>&1 | grep -E "tc profile|C[0-9] " | tail -2
done
echo "--- C3 with split forced on"
FSIL_TC_SPLIT=1 timeout 120 python tools/gpurun/gpurun_prof.py C3 2000000 2 2>&1 | grep -E "tc profile|C[0-9] " | tail -2
