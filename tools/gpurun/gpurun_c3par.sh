#!/bin/bash
cd "$GRAFT_REPO_ROOT"
cat > /tmp/c3par.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2303_14102_b200 import Context, datagen
ctx = Context(0)
for n in (20000, 50000):
    X, L, metric = datagen.generate_host("C3", n=n)
    ref = oracle.silhouette(X, L, metric)
    got = ctx.silhouette(X, L, metric)
    d = np.abs(got.s - ref.s)
    print(n, "dS=%.3e" % (got.mean - ref.mean), "max ds=%.3e" % d.max(), "sum(ds)/n=%.3e" % ((got.s - ref.s).sum() / n),
          "nb mism", int((got.neighbour != ref.neighbour).sum()), "stats", {k: ctx.stats()[k] for k in ("path", "agg_path", "flagged_rows", "exact_rows")})
PY
for lib in ab/libfsil_start.so paper_2303_14102_b200/libfsil.so; do echo "== $lib"; FSIL_LIB_PATH=$PWD/$lib timeout 300 python /tmp/c3par.py; done
