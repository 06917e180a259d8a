"""Builder debug tool: run random shapes through the C ABI with a per-shape verdict."""
import sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_14102_b200 import Context, datagen
import oracle
for spec in sys.argv[1:]:
    parts = spec.split(",")
    if parts[0] == "b":  # separated blobs
        n, d, k, metric = int(parts[1]), int(parts[2]), int(parts[3]), parts[4]
        rng = np.random.default_rng(n + d + k)
        centres = rng.normal(size=(k, d)) * 5.0
        L = rng.integers(0, k, n)
        X = (centres[L] + rng.normal(size=(n, d))).astype(np.float32)
    elif parts[0].startswith("C"):
        X, L, metric = datagen.generate_host(parts[0], n=int(parts[1]))
    else:
        n, d, k, metric = int(parts[0]), int(parts[1]), int(parts[2]), parts[3]
        rng = np.random.default_rng(n + d + k)
        X = (rng.normal(size=(n, d)) + rng.normal(size=(1, d)) * 3).astype(np.float32)
        L = rng.integers(0, k, n)
    ctx = Context(0)
    ctx.set_path(int(os.environ.get("DBG_PATH", "0")))
    try:
        got = ctx.silhouette(X, L, metric)
        ref = oracle.silhouette(X, L, metric)
        print(spec, "ok", got.mean - ref.mean, int((got.neighbour != ref.neighbour).sum()),
              float(np.abs(got.s - ref.s).max()), ctx.stats()["flagged_rows"], flush=True)
    except Exception as e:
        print(spec, "FAIL", e, flush=True)
        break
    ctx.close()
