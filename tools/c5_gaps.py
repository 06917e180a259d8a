"""Builder experiment (not product code): the C5 key-gap distribution, to size the neighbour
certificate.  Exact fp64 cosine keys 1 - (Omega_k . x/||x||)/n_k of a row sample against the
full-size aggregates; for each certificate width eps, how many rows have 1 / 2 / 3 / more
foreign clusters within 2*eps of their best (own excluded).

    python tools/c5_gaps.py [--rows 20000]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2303_14102_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=20000)
ap.add_argument("--out", default="gpurun_out/c5_gaps.json")
a = ap.parse_args()
Xd, Ld, metric = datagen.generate_device("C5")
X = Xd.cpu().numpy()
L = Ld.cpu().numpy()
del Xd, Ld
dense, raw = oracle.first_appearance(L)
k = raw.shape[0]
counts, sums, _ = oracle.aggregate_dense(X, dense, k, "cosine")
rows = np.random.default_rng(9).choice(X.shape[0], a.rows, replace=False)
x = X[rows].astype(np.float64)
xn = x / np.linalg.norm(x, axis=1, keepdims=True)
cross = xn @ sums.T                      # [rows, K]
keys = 1.0 - cross / counts[None, :]
keys[np.arange(a.rows), dense[rows]] = np.inf
keys.sort(axis=1)
gap = keys - keys[:, :1]
mu_norm = np.linalg.norm(sums / counts[:, None], axis=1)
res = {"rows": a.rows, "k": int(k), "mu_norm_max": float(mu_norm.max()), "mu_norm_median": float(np.median(mu_norm)),
       "gap2_quantiles": {q: float(np.quantile(gap[:, 1], q)) for q in (0.001, 0.01, 0.05, 0.1, 0.5)},
       "by_eps": {}}
for eps in (5e-5, 1e-4, 2e-4, 3.5e-4, 5e-4, 1e-3):
    within = (gap <= 2 * eps).sum(axis=1)  # includes the best itself
    res["by_eps"][str(eps)] = {f"ge{m}": float((within >= m).mean()) for m in (2, 3, 4, 5, 6, 9)}
print(json.dumps(res, indent=1))
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)
