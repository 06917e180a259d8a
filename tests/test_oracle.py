"""CPU tests of the oracle (the CPU restatement of the reference hot path) against
the reference's own known answers, its naive O(N^2 D) oracle, the
committed golden fixtures (scikit-learn) and SPEC.md's invariants.  These pin the
checker before it is trusted for GPU parity."""
import json
import os

import numpy as np
import pytest

import oracle

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def test_spec_square_sqeuclid():
    # every s_i = 15.5/16.5, mean 31/33
    X = np.array([[0, 0], [0, 1], [4, 0], [4, 1]], np.float32)
    for engine in ("fast", "naive"):
        r = oracle.silhouette(X, [1, 1, 2, 2], "sqeuclid", engine)
        assert np.allclose(r.a, 1.0) and np.allclose(r.b, 16.5)
        assert np.allclose(r.s, 15.5 / 16.5, rtol=0, atol=1e-15)
        assert abs(r.mean - 31 / 33) < 1e-15


def test_spec_orthogonal_cosine():
    # SPEC.md:213-214,221,461
    X = np.array([[1, 0], [2, 0], [0, 1], [0, 3]], np.float32)
    for engine in ("fast", "naive"):
        r = oracle.silhouette(X, [0, 0, 1, 1], "cosine", engine)
        assert np.allclose(r.s, 1.0) and r.mean == 1.0
        assert np.allclose(r.a, 0.0) and np.allclose(r.b, 1.0)


def test_spec_per_op_examples():
    assert abs(oracle.assemble_score(1.0, 16.5) - 15.5 / 16.5) < 1e-15
    assert oracle.assemble_score(0.0, 0.0) == 0.0
    assert oracle.assemble_score(2.0, 1.0) == -0.5
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.assemble_score(-1.0, 1.0)                                  # report.cpp:8-11
    assert [e - b for b, e in oracle.plan_shards(10, 3)] == [4, 3, 3]
    assert oracle.plan_shards(2, 8) == [(0, 1), (1, 2)]
    assert oracle.plan_shards(5, 1) == [(0, 5)]
    # partial stats / merge examples
    X = np.array([[0, 0], [0, 1], [4, 0]], np.float32)
    c, s, p = oracle.aggregate(X, [0, 0, 1], "sqeuclid")
    assert list(c) == [2, 1] and list(p) == [1.0, 16.0]
    assert s.tolist() == [[0.0, 1.0], [4.0, 0.0]]
    # Omega examples
    X = np.array([[1, 0], [2, 0], [0, 1], [0, 3]], np.float32)
    c, s, _ = oracle.aggregate(X, [0, 0, 1, 1], "cosine")
    assert s.tolist() == [[2.0, 0.0], [0.0, 2.0]]


def test_first_appearance_densify():
    # SPEC.md:60 ("b","a","b" -> [0,1,0]) with int labels (dataset.cpp:63-68)
    X = np.array([[0.0], [1.0], [0.5], [3.0]], np.float32)
    r = oracle.silhouette(X, [7, 3, 7, 3], "sqeuclid")
    assert r.own.tolist() == [0, 1, 0, 1] and r.dense_to_raw.tolist() == [7, 3]


@pytest.mark.parametrize("labels,msg", [([5, 5, 5], "single cluster"), ([1], "at least 2 points")])
def test_validation_errors(labels, msg):
    X = np.zeros((len(labels), 2), np.float32) + np.arange(len(labels))[:, None]
    with pytest.raises(oracle.OracleValidationError, match=msg):
        oracle.silhouette(X, labels)


def test_nonfinite_and_zero_norm():
    X = np.array([[0, 1], [1, np.nan], [2, 2]], np.float32)
    with pytest.raises(oracle.OracleValidationError, match="point 1, dimension 1"):
        oracle.silhouette(X, [0, 1, 1])
    X = np.array([[0, 1], [0, 0], [2, 2]], np.float32)
    with pytest.raises(oracle.OracleValidationError, match=r"zero vector \(point 1\)"):
        oracle.silhouette(X, [0, 1, 1], "cosine")
    with pytest.raises(oracle.OracleValidationError, match="no fast engine"):
        oracle.silhouette(X + 1, [0, 1, 1], "euclid")


def test_sklearn_goldens():
    for case in GOLDEN["sklearn_cases"]:
        X = np.array(case["X"], np.float32)
        r = oracle.silhouette(X, case["labels"], case["metric"])
        assert np.allclose(r.s, case["s"], rtol=1e-9, atol=1e-12)
        assert abs(r.mean - case["mean"]) < 1e-12


def _random_dataset(rng):
    n = int(rng.integers(4, 501))
    d = int(rng.integers(1, 17))
    k = int(rng.integers(2, 11))
    X = rng.normal(size=(n, d)) * rng.uniform(0.1, 5) + rng.normal(size=(1, d)) * 4
    L = rng.integers(0, k, n)
    L[: k] = np.arange(k)                       # every cluster present
    if rng.random() < 0.3:
        L[rng.integers(0, n)] = k              # singleton cluster
    if rng.random() < 0.3 and n > 3:
        X[1] = X[0]                             # duplicate points
    X = X.astype(np.float32)
    if np.any(np.linalg.norm(X, axis=1) == 0):
        X += 1.0
    return X, rng.permutation(L) * 3 + 1


def test_fast_equals_naive_property():
    # >= 200 seeded datasets, per-point rel 1e-9 / abs 1e-12, mean 1e-12
    rng = np.random.default_rng(460)
    for _ in range(200):
        X, L = _random_dataset(rng)
        for metric in ("sqeuclid", "cosine"):
            f = oracle.silhouette(X, L, metric, "fast")
            nv = oracle.silhouette(X, L, metric, "naive")
            for a, b in ((f.a, nv.a), (f.b, nv.b), (f.s, nv.s)):
                assert np.all(np.abs(a - b) <= 1e-12 + 1e-9 * np.abs(b))
            assert abs(f.mean - nv.mean) <= 1e-12
            assert np.array_equal(f.neighbour, nv.neighbour) or np.allclose(f.b, nv.b)


def test_invariants():
    # bounds, permutation, relabel, translation, positive scale, singleton
    rng = np.random.default_rng(464)
    for _ in range(20):
        X, L = _random_dataset(rng)
        r = oracle.silhouette(X, L, "sqeuclid")
        assert np.all(np.abs(r.s) <= 1.0)
        perm = rng.permutation(X.shape[0])
        rp = oracle.silhouette(X[perm], L[perm], "sqeuclid")
        assert np.allclose(rp.s, r.s[perm], atol=1e-12)
        rl = oracle.silhouette(X, L * 7 + 100, "sqeuclid")
        assert np.allclose(rl.s, r.s, atol=1e-15)
        rt = oracle.silhouette(X.astype(np.float64) + 3.0, L, "sqeuclid")
        assert np.allclose(rt.s, r.s, rtol=1e-9, atol=1e-9)
        c = oracle.silhouette(X, L, "cosine")
        cs = oracle.silhouette(X.astype(np.float64) * rng.uniform(0.5, 4, size=(X.shape[0], 1)), L, "cosine")
        assert np.allclose(cs.s, c.s, atol=1e-12)
        sizes = np.bincount(r.own)
        assert np.all(r.s[sizes[r.own] == 1] == 0.0)


def test_shard_independence_and_determinism():
    # SPEC.md:463 (W=4 bit-identical to W=1) and SPEC.md:466 (byte-identical reruns)
    rng = np.random.default_rng(463)
    X = rng.normal(size=(20000, 16)).astype(np.float32)
    L = rng.integers(0, 10, 20000)
    r1 = oracle.silhouette(X, L, "sqeuclid", shards=1)
    r4 = oracle.silhouette(X, L, "sqeuclid", shards=4)
    r4b = oracle.silhouette(X, L, "sqeuclid", shards=4)
    assert np.array_equal(r1.s, r4.s) and r1.mean == r4.mean
    assert np.array_equal(r4.s, r4b.s) and r4.mean == r4b.mean


def test_aggregate_dense_and_score_rows_agree_with_full_run():
    rng = np.random.default_rng(7)
    X = rng.normal(size=(3000, 9)).astype(np.float32)
    L = rng.integers(0, 13, 3000) * 11
    dense, raw = oracle.first_appearance(L)
    for metric in ("sqeuclid", "cosine"):
        full = oracle.silhouette(X, L, metric)
        assert raw.tolist() == full.dense_to_raw.tolist()
        c, s, p = oracle.aggregate_dense(X, dense, len(raw), metric)
        rows = np.arange(0, 3000, 13)
        a, b, sv, nb = oracle.score_rows(X, dense, c, s, p, rows, metric)
        assert np.array_equal(sv, full.s[rows]) and np.array_equal(nb, full.neighbour[rows])
