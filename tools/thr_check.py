"""Threshold-mode check (builder tool): shapes that take the threshold scan, against the
oracle (neighbour identical, s/S tight), with the per-call statistics.

    python tools/thr_check.py [--big]     # FSIL_TC_THR=0 in the environment: the old scan"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2303_14102_b200 import Context, datagen  # noqa: E402
from test_gpu_parity import check  # noqa: E402

ctx = Context(0)
rng = np.random.default_rng(5)


def blobs(n, d, k, spread, noise=1.0):
    cen = rng.normal(size=(k, d)) * spread
    lab = rng.integers(0, k, n)
    X = (cen[lab] + rng.normal(size=(n, d)) * noise).astype(np.float32)
    # nearest-centre labels: overlapping, uneven clusters (C4's recipe)
    if n * k <= 4e8:
        d2 = (X.astype(np.float64) ** 2).sum(1)[:, None] - 2 * X.astype(np.float64) @ cen.T + (cen ** 2).sum(1)[None]
        lab = d2.argmin(1)
    return X, lab


cases = [("overlap d32", *blobs(120_000, 32, 700, 1.0)), ("separated d32", *blobs(120_000, 32, 1000, 3.0)),
         ("d16", *blobs(150_000, 16, 600, 1.5)), ("d48", *blobs(100_000, 48, 300, 2.0)),
         ("k257", *blobs(80_000, 32, 257, 2.0)), ("offset", *blobs(100_000, 32, 500, 2.0))]
cases[-1] = ("offset", cases[-1][1] + np.float32(500.0), cases[-1][2])
for name, X, L in cases:
    t0 = time.time()
    got, ref = check(ctx, X, L, "sqeuclid", "tcgen05", label=name)
    st = ctx.stats()
    print(f"{name}: n={X.shape[0]} d={X.shape[1]} k={st['k']} thr={st['tc_threshold']} agg={st['agg_path']} "
          f"flagged={st['flagged_rows']} pairs={st['pair_rows']} S={got.mean:.12f} dS={abs(got.mean - ref.mean):.2e} "
          f"mism={int((got.neighbour != ref.neighbour).sum())} ({time.time() - t0:.1f}s)", flush=True)
for cfg, n in (("C4", 400_000),) + ((("C4", 4_000_000),) if "--big" in sys.argv else ()):
    X, L, metric = datagen.generate_host(cfg, n=n)
    got, ref = check(ctx, X, L, metric, "tcgen05", label=cfg)
    st = ctx.stats()
    print(f"{cfg}:{n} thr={st['tc_threshold']} flagged={st['flagged_rows']} pairs={st['pair_rows']} "
          f"dS={abs(got.mean - ref.mean):.2e} mism={int((got.neighbour != ref.neighbour).sum())}", flush=True)
print("thr_check ok")
