#!/bin/bash
# smoke(), the sharded protocol under torchrun (one rank) and the default bench.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5; echo "smoke rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/sharded.err | tail -1 | cut -c1-400; echo "sharded rc=$?"
