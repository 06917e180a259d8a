"""Generate the committed golden fixtures under tests/golden/.

Sources of truth (the reference ships no test vectors):
  * SPEC.md known answers (4-point square dataset -> mean 31/33; orthogonal
    cosine dataset -> mean 1; per-op examples) -- hand-derivable, written inline;
  * scikit-learn's silhouette_samples (metric "sqeuclidean" / "cosine"), an
    independent implementation with the same singleton (s = 0) and n-1
    own-cluster conventions, on small seeded datasets;
  * the reference's own blob generator recipe (blobs.hpp:13-44, blobs.cpp:11-54)
    restated in pure Python here (SplitMix64 + Box-Muller), for the C1 input.

Run:  python tests/golden/make_golden.py
"""
import json
import math
import os

import numpy as np
from sklearn.metrics import silhouette_samples

HERE = os.path.dirname(os.path.abspath(__file__))
MASK = (1 << 64) - 1


def splitmix64(seed):
    state = seed
    while True:
        state = (state + 0x9E3779B97F4A7C15) & MASK
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        yield z ^ (z >> 31)


def gaussian_stream(seed):
    rng = splitmix64(seed)
    while True:
        u1 = (next(rng) >> 11) * 2.0 ** -53
        u2 = (next(rng) >> 11) * 2.0 ** -53
        r = math.sqrt(-2.0 * math.log1p(-u1))
        th = 2.0 * math.pi * u2
        yield r * math.cos(th)
        yield r * math.sin(th)


def blobs(n, d, k, spread, separation, seed):
    g = gaussian_stream(seed)
    centres = [[separation * next(g) for _ in range(d)] for _ in range(k)]
    X = np.empty((n, d))
    L = np.empty(n, np.int32)
    for i in range(n):
        c = i % k
        L[i] = c
        for l in range(d):
            X[i, l] = centres[c][l] + spread * next(g)
    return X, L


def main():
    out = {}
    rng = np.random.default_rng(20230314)
    cases = []
    for idx in range(12):
        n = int(rng.integers(20, 300))
        d = int(rng.integers(1, 12))
        k = int(rng.integers(2, 8))
        X = rng.normal(size=(n, d)).astype(np.float32) * rng.uniform(0.5, 4)
        X += rng.normal(size=(1, d)).astype(np.float32) * 3
        L = rng.integers(0, k, n) * 5 - 7
        if idx % 3 == 0:  # a singleton cluster
            L[rng.integers(0, n)] = 999
        for metric in ("sqeuclidean", "cosine"):
            s = silhouette_samples(X.astype(np.float64), L, metric=metric)
            cases.append({"X": X.tolist(), "labels": L.tolist(), "metric":
                          "sqeuclid" if metric == "sqeuclidean" else "cosine",
                          "s": s.tolist(), "mean": float(s.mean())})
    out["sklearn_cases"] = cases
    Xb, Lb = blobs(64, 3, 4, 1.0, 8.0, 42)
    out["blobs_n64_d3_k4_seed42"] = {"X": Xb.tolist(), "labels": Lb.tolist()}
    out["spec_square"] = {"X": [[0, 0], [0, 1], [4, 0], [4, 1]], "labels": ["A", "A", "B", "B"],
                          "a": 1.0, "b": 16.5, "s": 15.5 / 16.5, "mean": 31 / 33}
    out["spec_cosine"] = {"X": [[1, 0], [2, 0], [0, 1], [0, 3]], "labels": ["A", "A", "B", "B"],
                          "s": 1.0, "mean": 1.0}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
