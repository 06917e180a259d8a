"""Small cases that reach every libfsil kernel variant, for compute-sanitizer
(tools/gpu/sanitize.sh: memcheck, racecheck, synccheck, initcheck).  Each case is
checked against the oracle so a sanitizer run is also a parity run.

  FFMA + batched aggregation (C1); tcgen05 three-group decoupled (C2); two-group
  in-place + label-sorted aggregation (C3); A-resident multi-block (C4 shape);
  streaming A scratch + top-3 pairs + tiled refinement (C5 shape); the fp64 path;
  the fp64 front end; the naive engine; the shard protocol with device exchange.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2303_14102_b200 import Context, datagen  # noqa: E402


def check(tag, got, ref):
    nb = int((got.neighbour != ref.neighbour).sum())
    ds = float(np.abs(got.s - ref.s).max())
    ok = nb == 0 and ds <= 1e-5 and abs(got.mean - ref.mean) <= 1e-6
    print(f"{tag}: {'ok' if ok else 'MISMATCH'} nb_mismatch={nb} max|ds|={ds:.2e}", flush=True)
    return ok


def main(which):
    ctx = Context(0)
    ok = True
    cases = [("C1", 4000, 1), ("C2", 4000, 2), ("C2", 4000, 1), ("C3", 3000, 2), ("C4", 3000, 2),
             ("C5", 600, 2), ("C3", 1500, 3)]
    for cfg, n, path in cases:
        if which and cfg not in which:
            continue
        X, L, metric = datagen.generate_host(cfg, n=n)
        ctx.set_path(path)
        ok &= check(f"{cfg} n={n} path={path}", ctx.silhouette(X, L, metric), oracle.silhouette(X, L, metric))
    ctx.set_path(0)
    if not which or "extra" in which:
        rng = np.random.default_rng(3)
        X = rng.standard_normal((1200, 20)) + 100.0
        L = rng.integers(0, 5, 1200)
        ok &= check("fp64 front end", ctx.silhouette(X, L, "sqeuclid"), oracle.silhouette(X, L, "sqeuclid"))
        X32 = X.astype(np.float32)
        ok &= check("naive", ctx.silhouette(X32, L, "cosine", _naive=True),
                    oracle.silhouette(X32, L, "cosine", engine="naive"))
        from paper_2303_14102_b200 import plan_shards
        import torch
        ref = oracle.silhouette(X32, L, "sqeuclid")
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
        from test_gpu_parity import _shard_loopback
        means, errors, s, nb, _ = _shard_loopback(X32, L, "sqeuclid", 3, 0, device_exchange=True)
        good = not errors and np.array_equal(nb, ref.neighbour) and np.abs(s - ref.s).max() <= 1e-5
        print(f"shard protocol: {'ok' if good else 'MISMATCH'}", flush=True)
        ok &= good
        del torch, plan_shards
    ctx.close()
    print("ALL OK" if ok else "FAILURES", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
