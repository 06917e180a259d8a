#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for rep in 1 2 3; do for v in 0 1; do FSIL_TC_EG3=$v timeout 200 python tools/gpurun/gpurun_ab.py C2 1000000 2>&1 | tail -1 | sed "s/^/eg3=$v /"; done; done
for v in 0 1; do FSIL_TC_EG3=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('eg3=$v bench', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
