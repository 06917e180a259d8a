#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for v in 0 1 0 1; do FSIL_PDL=$v timeout 300 python tools/gpurun/gpurun_phases.py C2 C1 2>&1 | sed "s/^/pdl=$v /"; done
for v in 0 1; do FSIL_PDL=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$v bench', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
