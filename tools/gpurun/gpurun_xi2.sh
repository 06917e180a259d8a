#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for lib in ab/libfsil_prev.so paper_2303_14102_b200/libfsil.so; do echo "== $lib"; FSIL_LIB_PATH=$PWD/$lib timeout 300 python /tmp/c3par.py 2>/dev/null || true; done
cat > /tmp/c3par.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2303_14102_b200 import Context, datagen
ctx = Context(0)
for cfg, n in (("C3", 20000), ("C3", 50000), ("C4", 30000), ("C5", 4000)):
    X, L, metric = datagen.generate_host(cfg, n=n)
    ref = oracle.silhouette(X, L, metric)
    got = ctx.silhouette(X, L, metric)
    d = np.abs(got.s - ref.s)
    print(cfg, n, "dS=%.3e" % (got.mean - ref.mean), "max ds=%.3e" % d.max(), "nb mism", int((got.neighbour != ref.neighbour).sum()),
          {k: ctx.stats()[k] for k in ("path", "agg_path", "flagged_rows", "exact_rows")}, flush=True)
PY
for lib in ab/libfsil_prev.so paper_2303_14102_b200/libfsil.so; do echo "== $lib"; FSIL_LIB_PATH=$PWD/$lib timeout 600 python /tmp/c3par.py; done
for c in "C3 2000000" "C4 2000000" "C5 200000"; do
for lib in ab/libfsil_prev.so paper_2303_14102_b200/libfsil.so; do FSIL_LIB_PATH=$PWD/$lib timeout 300 python tools/gpurun/gpurun_ab.py $c 2>&1 | tail -1; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
