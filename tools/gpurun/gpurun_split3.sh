#!/bin/bash
cd "$GRAFT_REPO_ROOT"
cat > /tmp/c3par.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import oracle
from paper_2303_14102_b200 import Context, datagen
ctx = Context(0)
for cfg, n in (("C3", 20000), ("C3", 50000), ("C4", 30000)):
    X, L, metric = datagen.generate_host(cfg, n=n)
    ref = oracle.silhouette(X, L, metric)
    got = ctx.silhouette(X, L, metric)
    print(cfg, n, "dS=%.3e" % (got.mean - ref.mean), "max ds=%.3e" % np.abs(got.s - ref.s).max(), "mean ds=%.3e" % (got.s - ref.s).mean(), flush=True)
PY
for sp in 0 1; do echo "split=$sp"; FSIL_TC_SPLIT=$sp timeout 600 python /tmp/c3par.py 2>&1 | head -3; FSIL_TC_SPLIT=$sp timeout 300 python tools/gpurun/gpurun_ab.py C3 2000000 2>&1 | tail -1; done
