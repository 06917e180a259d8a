"""GPU parity: libfsil (through the C ABI) against the CPU oracle on the same
seeded inputs.  Bar (BASELINE.json north_star): identical neighbour cluster
(dense id, reference tie rule), |ds_i| <= 1e-5, |dS| <= 1e-6; a_i / b_i within
1e-4 relative (AB_RTOL; not a BASELINE bar).  Runs on a B200 under gpurun
(`pytest -m gpu`)."""
import json
import math
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

S_TOL, MEAN_TOL = 1e-5, 1e-6
AB_RTOL = 1e-4
# Every fast path computes a_i, b_i, s_i in fp64 with the reference formulas (the
# tensor-core pass only nominates the neighbour; the exact pass recomputes every row), so
# the achieved agreement is fp64 summation-order noise, asserted far inside the bars:
S_TIGHT, MEAN_TIGHT, AB_TIGHT = 1e-9, 1e-10, 1e-9
PATHS = {"auto": 0, "ffma": 1, "tcgen05": 2, "fp64": 3}


@pytest.fixture(scope="module")
def ctx():
    from paper_2303_14102_b200 import Context
    c = Context(0)
    yield c
    c.close()


def reference_noise_ties(X, ref, metric, rows, alt):
    raw = np.asarray(ref.dense_to_raw)[ref.own]  # same first-appearance order as ref
    counts, sums, psi = oracle.aggregate(X, raw, metric)
    x = X[rows].astype(np.float64)
    out = []
    for i, r in enumerate(rows):
        vals, scales = [], []
        for k in (ref.neighbour[r], alt[i]):
            n = float(counts[k])
            cross = float(sums[k] @ x[i])
            if metric == "cosine":
                nrm = np.sqrt(x[i] @ x[i])
                vals.append(min(max(1.0 - cross / nrm / n, 0.0), 2.0))
                scales.append(1.0 + abs(cross / nrm / n))
            else:
                xi = float(x[i] @ x[i])
                vals.append(max(0.0, xi + psi[k] / n - 2.0 * cross / n))
                scales.append(xi + psi[k] / n + 2.0 * abs(cross) / n)
        out.append(abs(vals[0] - vals[1]) <= 1e-12 * max(scales))
    return np.array(out)


def check(ctx, X, L, metric, path="auto", label=""):
    ctx.set_path(PATHS[path])
    got = ctx.silhouette(X, L, metric)
    ref = oracle.silhouette(X, L, metric)
    tag = f"{label} {metric} path={path} n={X.shape[0]} d={X.shape[1]}"
    assert got.cluster_names == ref.dense_to_raw.tolist(), tag
    assert np.array_equal(got.own, ref.own), tag
    mism = np.flatnonzero(got.neighbour != ref.neighbour)
    if mism.size:
        # Only rows whose two candidates tie within the fp64 rounding noise of the
        # reference formula itself (terms of size xi + Psi/n + 2|cross|/n) may
        # differ: there the reference's own choice depends on its summation order.
        ties = reference_noise_ties(X, ref, metric, mism, got.neighbour[mism])
        assert ties.all(), (f"{tag}: {int((~ties).sum())} certain-neighbour mismatches, "
                            f"rows {mism[~ties][:5]}")
        assert mism.size <= max(2, X.shape[0] // 20), tag
    assert np.abs(got.s - ref.s).max() <= S_TOL, tag
    assert abs(got.mean - ref.mean) <= MEAN_TOL, tag
    for g, r in ((got.a, ref.a), (got.b, ref.b)):
        assert np.all(np.abs(g - r) <= AB_RTOL * np.maximum(1.0, np.abs(r))), tag
    if True:
        # fp64 everywhere: summation-order noise only (amplified by the squared-Euclidean
        # cancellation n xi + Psi - 2 cross when ||x|| >> the cluster spread)
        amp = 1.0
        if metric == "sqeuclid":
            xi = (X.astype(np.float64) ** 2).sum(1)
            pos = ref.b > 0
            if pos.any():
                amp = min(1e6, 1.0 + 1e-3 * float(np.max(xi[pos] / ref.b[pos])))
        assert np.abs(got.s - ref.s).max() <= S_TIGHT * amp, (tag, np.abs(got.s - ref.s).max())
        assert abs(got.mean - ref.mean) <= MEAN_TIGHT * amp, (tag, abs(got.mean - ref.mean))
        for g, r in ((got.a, ref.a), (got.b, ref.b)):
            assert np.all(np.abs(g - r) <= AB_TIGHT * amp * np.maximum(1.0, np.abs(r))), tag
    ctx.set_path(0)
    return got, ref


def test_spec_goldens(ctx):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
    sq = g["spec_square"]
    got = ctx.silhouette(np.array(sq["X"], np.float32), [1, 1, 2, 2], "sqeuclid")
    assert np.allclose(got.s, sq["s"], atol=1e-15) and abs(got.mean - 31 / 33) < 1e-15
    assert np.allclose(got.a, 1.0) and np.allclose(got.b, 16.5)
    cs = g["spec_cosine"]
    got = ctx.silhouette(np.array(cs["X"], np.float32), [0, 0, 1, 1], "cosine")
    assert np.allclose(got.s, 1.0) and got.mean == 1.0


def test_sklearn_goldens(ctx):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
    for case in g["sklearn_cases"]:
        got = ctx.silhouette(np.array(case["X"], np.float32), case["labels"], case["metric"])
        assert np.abs(got.s - np.array(case["s"])).max() <= 1e-9
        assert abs(got.mean - case["mean"]) <= 1e-12


SHAPES = [(500, 5, 6), (1000, 16, 8), (3000, 64, 20), (777, 3, 3), (2000, 33, 40), (5000, 128, 100),
          (2500, 7, 32), (4000, 1, 5), (3000, 100, 2), (1500, 200, 300)]


@pytest.mark.parametrize("n,d,k", SHAPES)
@pytest.mark.parametrize("metric", ["sqeuclid", "cosine"])
def test_random_shapes(ctx, n, d, k, metric):
    rng = np.random.default_rng(n * 31 + d * 7 + k)
    X = (rng.normal(size=(n, d)) + rng.normal(size=(1, d)) * 3).astype(np.float32)
    L = rng.integers(0, k, n) * 7 - 3
    check(ctx, X, L, metric)


@pytest.mark.parametrize("path", ["ffma", "fp64"])
@pytest.mark.parametrize("metric", ["sqeuclid", "cosine"])
def test_paths_agree(ctx, path, metric):
    rng = np.random.default_rng(5)
    X = rng.normal(size=(4096, 48)).astype(np.float32)
    L = rng.integers(0, 24, 4096)
    check(ctx, X, L, metric, path)


def test_edge_singleton_and_pairs(ctx):
    rng = np.random.default_rng(11)
    X = rng.normal(size=(600, 8)).astype(np.float32)
    L = rng.integers(0, 5, 600)
    L[17] = 50          # singleton: a = 0, s = 0, b and neighbour still reported
    L[[3, 400]] = 60    # size-2 cluster
    for metric in ("sqeuclid", "cosine"):
        got, ref = check(ctx, X, L, metric)
        assert got.s[17] == 0.0 and got.a[17] == 0.0 and got.b[17] > 0


def test_edge_duplicates_across_clusters(ctx):
    # coincident points in two clusters: a = b = 0 -> s = 0 (report.cpp:12)
    X = np.array([[1, 2], [1, 2], [1, 2], [1, 2], [5, 5], [5, 6]], np.float32)
    L = [0, 0, 1, 1, 2, 2]
    got, _ = check(ctx, X, L, "sqeuclid")
    assert np.all(got.s[:4] == 0.0)


def test_edge_exact_tie_lowest_dense_id(ctx):
    # two identical foreign clusters: neighbour = lowest dense id (strict <)
    base = np.array([[0, 0], [0.1, 0], [0, 0.1]], np.float32)
    far = base + np.float32(10)
    X = np.concatenate([far, base, far])   # raw labels 9 (far), 4 (base), 7 (far copy)
    L = [9, 9, 9, 4, 4, 4, 7, 7, 7]
    for metric in ("sqeuclid", "cosine"):
        got, ref = check(ctx, X + np.float32(1), L, metric)
        assert got.neighbour[3] == 0  # dense id of raw 9, not 7


def test_edge_first_appearance_not_numeric(ctx):
    rng = np.random.default_rng(3)
    X = rng.normal(size=(300, 4)).astype(np.float32)
    L = rng.choice([2**31 - 1, -2**31, 0, 17, -5], size=300)
    got, ref = check(ctx, X, L, "sqeuclid")
    assert got.cluster_names[0] == int(L[0])


def test_edge_k2_and_many_labels(ctx):
    rng = np.random.default_rng(4)
    X = rng.normal(size=(3000, 6)).astype(np.float32)
    check(ctx, X, rng.integers(0, 2, 3000), "sqeuclid")
    # K close to N: hash-table growth path, mostly singletons
    L = rng.integers(0, 2500, 3000) * 9973
    check(ctx, X, L, "cosine")


def test_edge_negative_cancellation_clamp(ctx):
    # A cluster of identical points far from the origin: its own-cluster mean is
    # exactly 0 in real arithmetic, and the reference formula's cancellation
    # (n*xi + Psi - 2*cross) can round to a tiny negative that max(0, .) clamps
    # (squared_euclidean.cpp:77,81).  Other clusters keep the fp64 noise small
    # relative to their distances, so the comparison stays meaningful.
    rng = np.random.default_rng(8)
    X = (np.float32(40) + rng.normal(size=(2000, 12)) * 2).astype(np.float32)
    L = rng.integers(0, 4, 2000)
    X[L == 2] = X[np.flatnonzero(L == 2)[0]]
    for metric in ("sqeuclid", "cosine"):
        got, ref = check(ctx, X, L, metric)
        assert np.all(got.a >= 0) and np.all(got.b >= 0)
        xi = (X[L == 2][0].astype(np.float64) ** 2).sum()
        assert np.all(got.a[L == 2] <= 1e-12 * xi)


def _blobs(n, d, k, seed, spread=5.0):
    rng = np.random.default_rng(seed)
    centres = rng.normal(size=(k, d)) * spread
    L = rng.integers(0, k, n)
    X = (centres[L] + rng.normal(size=(n, d))).astype(np.float32)
    return X, L


@pytest.mark.parametrize("nstg", ["2", "3", "4", ""])
@pytest.mark.parametrize("n,d,k,metric", [(40000, 256, 200, "sqeuclid"), (40000, 256, 200, "cosine"),
                                          (45000, 768, 300, "cosine")])
def test_tc_streaming_stage_counts(ctx, monkeypatch, nstg, n, d, k, metric):
    """The A-scratch streaming mode (several cluster blocks whose K chunks outnumber the X
    stages) with several tiles per CTA, across X-stage counts: every (stages, chunks,
    passes) combination must keep the staging ring's barrier phases in step.  Separated
    blobs, so most neighbours are certified straight from the tensor-core pass and a
    misread stage would show up as a wrong neighbour, not only as a flagged row."""
    if nstg:
        monkeypatch.setenv("FSIL_TC_NSTG", nstg)
    X, L = _blobs(n, d, k, seed=n + d + k)
    got, ref = check(ctx, X, L, metric, "tcgen05", label=f"nstg={nstg or 'auto'}")
    assert ctx.stats()["flagged_rows"] < n // 2


@pytest.mark.parametrize("n,d,k,metric", [(30000, 200, 600, "cosine"), (30000, 136, 513, "sqeuclid"),
                                          (20000, 768, 1000, "sqeuclid"), (9000, 320, 2100, "cosine"),
                                          (3000, 192, 257, "cosine")])
def test_tc_pair_kernel_shapes(ctx, n, d, k, metric):
    """The CTA-pair kernel (score_tc2.cu) on streaming tables: a partial last K chunk
    (D = 200, 136: the second fp32 box absent, the MMA's K steps stop early), K not a
    multiple of the 256-column block (padding columns at +inf), an odd number of 128-row
    tiles (the peer CTA of the last pair idle), several super-tiles per pair."""
    X, L = _blobs(n, d, k, seed=n + d + k)
    check(ctx, X, L, metric, "tcgen05", label="pair")
    assert ctx.stats()["flagged_rows"] < n // 2


def test_tc_cosine_mixed_norms_unit_scale(ctx):
    """Cosine is invariant to per-point scaling, so rows scaled by 1e-3..1e-5 are valid
    input.  On the three-group kernel (BN = 32, batched aggregation) the x operand is not
    scaled (unit scale when max|x| is in [0.5, 2^14)), so those rows' fp16 pieces sit in
    the subnormal range: their dot error is absolute in x and the certificate has to
    charge it per row (floor_x / ||x||), not per the shard's largest element."""
    from paper_2303_14102_b200 import datagen
    X, L, metric = datagen.generate_host("C2", n=200_000)
    rng = np.random.default_rng(4)
    small = rng.choice(X.shape[0], 20_000, replace=False)
    X[small] *= (10.0 ** rng.uniform(-5, -3, small.size)).astype(np.float32)[:, None]
    got, ref = check(ctx, X, L, metric, "tcgen05", label="mixed norms")
    assert np.array_equal(got.neighbour[small], ref.neighbour[small])


def _nearest_centre_blobs(n, d, k, spread, seed, offset=0.0):
    """Gaussian blobs relabelled by nearest centre: overlapping, uneven clusters (C4's recipe)."""
    rng = np.random.default_rng(seed)
    cen = rng.normal(size=(k, d)) * spread
    X = (cen[rng.integers(0, k, n)] + rng.normal(size=(n, d))).astype(np.float32)
    x64 = X.astype(np.float64)
    d2 = (x64 ** 2).sum(1)[:, None] - 2 * x64 @ cen.T + (cen ** 2).sum(1)[None]
    return X + np.float32(offset), d2.argmin(1)


@pytest.mark.parametrize("name,n,d,k,spread,offset", [
    ("overlap d32", 120_000, 32, 700, 1.0, 0.0),     # heavy overlap: many rows with 2-4 candidates (three groups)
    ("separated d32", 120_000, 32, 1000, 3.0, 0.0),  # C4-like: almost every row certified outright
    ("d16", 150_000, 16, 600, 1.5, 0.0),             # one K step + the threshold step
    ("d48", 100_000, 48, 300, 2.0, 0.0),             # two fp32 boxes, 32 KB stages, B ring
    ("k257", 80_000, 32, 257, 2.0, 0.0),             # one column into the third cluster block
    ("k1200", 50_000, 32, 1200, 2.0, 0.0),           # resident table, no room for the third group's stages: two groups
    ("k2100", 40_000, 32, 2100, 2.0, 0.0),           # table too large to stay resident: B ring
    ("offset", 100_000, 32, 500, 2.0, 500.0),        # ||x|| >> spread: no row certifies, all refined
])
def test_tc_threshold_mode(ctx, name, n, d, k, spread, offset):
    """Threshold mode of the single-CTA tcgen05 kernel (sqeuclid, D <= 48, several cluster
    blocks, label-sorted aggregation): the comparison against the per-row certified threshold
    runs inside the MMA and the epilogue harvests sign bits.  Every row's neighbour must be
    the oracle's (candidate rows are resolved in fp64), a/b/s at fp64 noise."""
    X, L = _nearest_centre_blobs(n, d, k, spread, seed=5 + d + k, offset=offset)
    got, ref = check(ctx, X, L, "sqeuclid", "tcgen05", label=name)
    st = ctx.stats()
    assert st["tc_threshold"] == 1, (name, st)
    if offset == 0.0:
        assert st["flagged_rows"] < n // 4, (name, st)


def test_tc_threshold_mode_switch(ctx):
    """FSIL_THR_BRES / FSIL_THR_L1 are read once per process, so the ring variants are covered
    by shapes (d48, k2100 above); here: the threshold scan and the classic scan agree row for
    row on the same input (the classic scan is what K <= 128 or D > 48 shapes take)."""
    X, L = _nearest_centre_blobs(90_000, 32, 400, 2.0, seed=77)
    got, _ = check(ctx, X, L, "sqeuclid", "tcgen05", label="thr")
    assert ctx.stats()["tc_threshold"] == 1
    X2 = np.concatenate([X, np.zeros((X.shape[0], 32), np.float32)], axis=1)  # D = 64: classic scan
    got2, _ = check(ctx, X2, L, "sqeuclid", "tcgen05", label="classic")
    assert ctx.stats()["tc_threshold"] == 0
    assert np.array_equal(got.neighbour, got2.neighbour)
    assert np.abs(got.s - got2.s).max() <= 1e-12


@pytest.mark.parametrize("metric", ["sqeuclid", "cosine"])
@pytest.mark.parametrize("k_pad,d", [(0, 64), (97, 64), (290, 64), (290, 256), (290, 32), (290, 48)])
def test_tc_certificate_adversarial_near_ties(ctx, metric, k_pad, d):
    """Pins the neighbour certificate: rows placed at controlled distances from the
    bisector of two mirror clusters A (dense id 1) and B (dense id 2), so their top-2 gap
    runs log-uniformly from ~1e-10 to ~1e-1 relative -- across the tensor-core error bound --
    far from the origin (large ||x||, the dot-error regime).  Rows the certificate passes
    must carry exactly the oracle's neighbour; the rest go to the fp64 refinement.
    k_pad far-away clusters add cluster blocks (BN = 128, several blocks); at D = 256 the
    table is large enough for the top-3 epilogue, whose certified pairs must agree too."""
    rng = np.random.default_rng(17 + k_pad + d)
    base = np.full(d, 30.0) if metric == "sqeuclid" else np.zeros(d)
    e = np.zeros(d)
    e[0] = 1.0
    u = np.zeros(d)
    u[1] = 1.0
    off = 3.0
    if metric == "cosine":  # directions: A, B mirror about u; rows near u
        base = u * 10.0
    # mirror clusters: symmetric members so the means are exactly base +/- off*e
    def mirror(centre, m):
        v = rng.normal(size=(m // 2, d)) * 0.5
        return np.concatenate([centre + v, centre - v])
    A = mirror(base + off * e + 4.0 * u, 400)
    B = mirror(base - off * e + 4.0 * u, 400)
    n_rows = 30_000
    t = np.exp(rng.uniform(np.log(1e-9), np.log(1.0), n_rows)) * rng.choice([-1.0, 1.0], n_rows)
    rows = base + rng.normal(size=(n_rows, d)) * 0.3
    rows[:, 0] = base[0] + t  # signed distance from the (mirror) bisector
    parts, labels = [rows, A, B], [np.zeros(n_rows, int), np.ones(400, int), np.full(400, 2)]
    if k_pad:
        far = rng.normal(size=(k_pad, d)) * 3 + (200.0 if metric == "sqeuclid" else -50.0) * u
        parts.append(np.repeat(far, 3, axis=0) + rng.normal(size=(3 * k_pad, d)) * 0.1)
        labels.append(np.repeat(np.arange(3, 3 + k_pad), 3))
    X = np.concatenate(parts).astype(np.float32)
    L = np.concatenate(labels)
    got, ref = check(ctx, X, L, metric, "tcgen05", label=f"near ties k_pad={k_pad}")
    assert np.array_equal(got.neighbour[:n_rows], ref.neighbour[:n_rows])
    # both candidates really occur, and a good share of rows is decided on the fast pass
    assert set(np.unique(ref.neighbour[:n_rows])) >= {1, 2}
    assert ctx.stats()["flagged_rows"] < n_rows
    if metric == "sqeuclid" and d <= 48:  # the threshold scan (comparison inside the MMA)
        assert ctx.stats()["tc_threshold"] == 1


def test_tc_threshold_mode_edge_cases(ctx):
    """The reference's edge cases on the threshold scan (D = 32, K > 256): singleton clusters
    (s = 0, report.cpp:18-21), a two-point cluster, exact duplicates of other rows, a cluster of
    identical points (a = 0), and two clusters with identical members under different labels --
    every row's distance to them ties exactly, so the lowest dense id must win
    (squared_euclidean.cpp:94-103) wherever one of them is the neighbour."""
    X, L = _nearest_centre_blobs(60_000, 32, 300, 3.0, seed=91)
    L = L.astype(np.int64)
    rng = np.random.default_rng(92)
    extra_x, extra_l = [], []
    nxt = int(L.max()) + 1
    for _ in range(3):  # singletons, far from and close to other clusters
        extra_x.append(X[rng.integers(0, X.shape[0])][None] + rng.normal(size=(1, 32)).astype(np.float32) * 0.5)
        extra_l.append([nxt])
        nxt += 1
    extra_x.append(X[:2] + np.float32(0.25))  # a two-point cluster
    extra_l.append([nxt, nxt])
    nxt += 1
    dup = rng.choice(X.shape[0], 500, replace=False)  # exact duplicates keep their labels
    extra_x.append(X[dup])
    extra_l.append(L[dup])
    extra_x.append(np.repeat(X[7][None] + np.float32(1.0), 40, axis=0))  # identical points
    extra_l.append([nxt] * 40)
    nxt += 1
    twin = X[L == L[11]][:200] + np.float32(0.5)  # twin clusters: the same members twice
    extra_x += [twin, twin]
    extra_l += [[nxt] * twin.shape[0], [nxt + 1] * twin.shape[0]]
    X = np.concatenate([X] + extra_x).astype(np.float32)
    L = np.concatenate([L] + [np.asarray(e, np.int64) for e in extra_l])
    got, ref = check(ctx, X, L, "sqeuclid", "tcgen05", label="thr edge")
    assert ctx.stats()["tc_threshold"] == 1
    assert np.array_equal(got.neighbour, ref.neighbour)
    single = np.isin(L, np.arange(int(L.max()) - 6, int(L.max()) - 3))
    assert single.sum() == 3 and np.all(got.s[single] == 0.0) and np.all(got.a[single] == 0.0)
    # rows whose neighbour is a twin carry the lower of the two dense ids
    t0, t1 = np.flatnonzero(np.asarray(ref.dense_to_raw) == nxt)[0], np.flatnonzero(np.asarray(ref.dense_to_raw) == nxt + 1)[0]
    assert np.any(got.neighbour == min(t0, t1))
    other = ~np.isin(got.own, [t0, t1])
    assert not np.any(got.neighbour[other] == max(t0, t1))


def test_validation_errors_match_reference(ctx):
    from paper_2303_14102_b200 import ValidationError
    X = np.array([[0, 1], [1, np.nan], [2, 2], [3, 3]], np.float32)
    with pytest.raises(ValidationError, match="non-finite feature value at point 1, dimension 1"):
        ctx.silhouette(X, [0, 1, 1, 0], "sqeuclid")
    X = np.array([[0, 1], [0, 0], [2, 2], [3, 3]], np.float32)
    with pytest.raises(ValidationError, match=r"cosine distance undefined for zero vector \(point 1\)"):
        ctx.silhouette(X, [0, 1, 1, 0], "cosine")
    with pytest.raises(ValidationError, match="need K >= 2, got K = 1"):
        ctx.silhouette(X + 1, [3, 3, 3, 3], "sqeuclid")
    with pytest.raises(ValidationError, match="at least 2 points"):
        ctx.silhouette(np.ones((1, 3), np.float32), [0], "sqeuclid")
    with pytest.raises(ValidationError, match="no fast engine for plain euclidean"):
        ctx.silhouette(X + 1, [0, 1, 1, 0], "euclid")
    # NaN takes precedence over K < 2 (dataset.cpp:35 before :53)
    Xn = np.array([[0, 1], [np.inf, 1]], np.float32)
    with pytest.raises(ValidationError, match="non-finite"):
        ctx.silhouette(Xn, [1, 1], "sqeuclid")
    # the context stays usable after errors
    check(ctx, np.random.default_rng(0).normal(size=(100, 3)).astype(np.float32),
          np.arange(100) % 3, "sqeuclid")


# The two-phase batched aggregation (agg path 3) takes D in {16, 32, 64, 128} with small
# K*D: batches of 32 (D < 64) or 16 rows, partial last batches, fewer rows than one batch,
# Psi as an extra accumulated pair (squared Euclidean), and -- on the cosine tcgen05 path --
# the per-row ||x||^2 it hands to the scoring kernel.
@pytest.mark.parametrize("n,d,k", [(1003, 32, 12), (517, 128, 9), (10, 64, 3), (33, 16, 2), (4099, 64, 31),
                                   (20000, 32, 5)])
@pytest.mark.parametrize("metric", ["sqeuclid", "cosine"])
def test_batched_aggregation_shapes(ctx, n, d, k, metric):
    rng = np.random.default_rng(n + 11 * d + k)
    X = (rng.normal(size=(n, d)) + rng.normal(size=(1, d)) * 2).astype(np.float32)
    L = rng.integers(0, k, n) * 3 + 5
    got, _ = check(ctx, X, L, metric)
    assert ctx.stats()["agg_path"] == 3, "expected the batched aggregation path"
    # also through the tensor-core scoring kernel: decoupled mode with external ||x||^2 and
    # three epilogue groups at BN = 32 (D = 16: the second box absent; D = 128: two chunks)
    check(ctx, X, L, metric, "tcgen05")


def test_batched_aggregation_validation(ctx):
    """Validation inside the batched path (D = 64): the first non-finite element in
    row-major order wins (dataset.cpp:35-37); a zero row fails cosine (cos.cpp:119-123)."""
    from paper_2303_14102_b200 import ValidationError
    rng = np.random.default_rng(3)
    X = rng.normal(size=(300, 64)).astype(np.float32)
    L = np.arange(300) % 4
    Xb = X.copy()
    Xb[211, 40] = np.inf
    Xb[37, 5] = np.nan
    Xb[37, 63] = np.nan
    with pytest.raises(ValidationError, match="non-finite feature value at point 37, dimension 5"):
        ctx.silhouette(Xb, L, "sqeuclid")
    Xz = X.copy()
    Xz[150] = 0.0
    Xz[290] = 0.0
    with pytest.raises(ValidationError, match=r"cosine distance undefined for zero vector \(point 150\)"):
        ctx.silhouette(Xz, L, "cosine")
    got, _ = check(ctx, X, L, "cosine")  # still usable
    assert ctx.stats()["agg_path"] == 3


def test_determinism(ctx):
    rng = np.random.default_rng(9)
    X = rng.normal(size=(50000, 24)).astype(np.float32)
    L = rng.integers(0, 12, 50000)
    r1 = ctx.silhouette(X, L, "cosine")
    r2 = ctx.silhouette(X, L, "cosine")
    assert np.array_equal(r1.s, r2.s) and r1.mean == r2.mean and np.array_equal(r1.neighbour, r2.neighbour)


def test_determinism_batched_tcgen05_and_timing(ctx):
    """The C2-shaped path (batched aggregation, decoupled tcgen05 scoring, PDL chain):
    bit-identical across calls, and the per-phase timers (bench.py's roofline input)
    report the scoring kernel alone inside the scoring phase."""
    rng = np.random.default_rng(21)
    X = (rng.normal(size=(60000, 64)) + rng.normal(size=(1, 64))).astype(np.float32)
    L = rng.integers(0, 20, 60000)
    ctx.set_path(PATHS["tcgen05"])
    r1 = ctx.silhouette(X, L, "cosine")
    ctx.set_timing(True)
    r2 = ctx.silhouette(X, L, "cosine")
    st = ctx.stats()
    ctx.set_timing(False)
    ctx.set_path(0)
    assert np.array_equal(r1.s, r2.s) and r1.mean == r2.mean and np.array_equal(r1.neighbour, r2.neighbour)
    assert st["agg_path"] == 3 and st["path"] == PATHS["tcgen05"]
    assert 0.0 < st["ms_score_kernel"] <= st["ms_score"]
    assert all(st[k] > 0.0 for k in ("ms_densify", "ms_aggregate", "ms_refine"))


def _config(ctx, name, n=None):
    from paper_2303_14102_b200 import datagen
    X, L, metric = datagen.generate_host(name, n=n)
    return X, L, metric


def test_c1_full_and_naive_rows(ctx):
    X, L, metric = _config(ctx, "C1")
    got, ref = check(ctx, X, L, metric, label="C1")
    # naive O(N^2 D) definition (naive.cpp:30-71) on sampled rows, all N points
    rows = np.random.default_rng(1).choice(X.shape[0], 64, replace=False)
    X64 = X.astype(np.float64)
    sizes = np.bincount(got.own)
    for i in rows:
        dist = ((X64 - X64[i]) ** 2).sum(1)
        sums = np.bincount(got.own, dist, minlength=sizes.shape[0])
        own = got.own[i]
        a = sums[own] / (sizes[own] - 1)
        means = sums / sizes
        means[own] = np.inf
        nb = int(np.argmin(means))
        b = means[nb]
        s = 1 - a / b if a <= b else b / a - 1
        assert nb == got.neighbour[i] and abs(s - got.s[i]) <= 1e-9


def test_c2_full(ctx):
    X, L, metric = _config(ctx, "C2")
    check(ctx, X, L, metric, label="C2")


@pytest.mark.parametrize("name,n", [("C3", 400_000), ("C4", 400_000), ("C5", 20_000)])
def test_scaled_configs_full_oracle(ctx, name, n):
    X, L, metric = _config(ctx, name, n)
    check(ctx, X, L, metric, label=name)


def _full_size_gpu(ctx, name, path=0, data=None):
    """One full-size config on the device through fsil_silhouette_device -> host arrays.
    data=(Xd, Ld, metric) reuses already generated device inputs."""
    import torch
    from paper_2303_14102_b200 import datagen
    Xd, Ld, metric = data if data is not None else datagen.generate_device(name)
    n, d = Xd.shape
    s = torch.empty(n, dtype=torch.float64, device="cuda")
    nb = torch.empty(n, dtype=torch.int32, device="cuda")
    own = torch.empty(n, dtype=torch.int32, device="cuda")
    d2r = np.empty(min(n, 10_000_000), np.int32)
    ctx.set_path(path)
    try:
        mean, k = ctx.silhouette_device(Xd, Ld, metric, s=s, neighbour=nb, own=own, dense_to_raw=d2r)
        mean2, _ = ctx.silhouette_device(Xd, Ld, metric, s=s, neighbour=nb)
    finally:
        ctx.set_path(0)
    assert mean2 == mean  # bit-identical rerun
    out = dict(X=Xd, L=Ld, metric=metric, mean=mean, k=k, s=s.cpu().numpy(), nb=nb.cpu().numpy(),
               own=own.cpu().numpy(), d2r=d2r[:k].copy())
    s_h, nb_h, own_h = out["s"], out["nb"], out["own"]
    assert np.all(np.abs(s_h) <= 1.0) and abs(s_h.mean() - mean) <= 1e-9
    assert np.all(nb_h != own_h) and nb_h.min() >= 0 and nb_h.max() < k
    return out


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_oracle_all_rows(ctx, name):
    """BASELINE.json full sizes (C3: 1e7 x 128, K=100; C4: 1e8 x 32, K=1000) against the
    oracle on EVERY row: the oracle aggregates all N rows (engine.hpp:50-80 block plan
    and fold) and scores all N rows (score_range, sqE.cpp:84-108) on every host core.
    Bar: neighbours identical, |ds_i| <= 1e-5, |dS| <= 1e-6 -- and, because every s_i is
    computed in fp64 by the reference formulas, the achieved agreement is asserted
    at fp64 noise (|dS| <= 1e-10)."""
    g = _full_size_gpu(ctx, name)
    X, L = g["X"].cpu().numpy(), g["L"].cpu().numpy()
    del g["X"], g["L"]
    n = X.shape[0]
    dense, raw = oracle.first_appearance(L)
    del L
    assert raw.tolist() == g["d2r"].tolist() and np.array_equal(dense, g["own"])
    counts, sums, psi = oracle.aggregate_dense(X, dense, g["k"], g["metric"])
    _, _, sv, nbv = oracle.score_rows(X, dense, counts, sums, psi, None, g["metric"], threads=0, want_ab=False)
    mism = np.flatnonzero(nbv != g["nb"])
    assert mism.size == 0, f"{name}: {mism.size} neighbour mismatches, rows {mism[:5]}"
    ds = np.abs(sv - g["s"]).max()
    dS = abs(math.fsum(sv) / n - g["mean"])
    print(f"{name} full size: N={n} S_gpu={g['mean']:.15f} S_oracle={math.fsum(sv) / n:.15f} "
          f"|dS|={dS:.3e} max|ds_i|={ds:.3e}")
    assert ds <= S_TOL and dS <= MEAN_TOL
    assert ds <= S_TIGHT and dS <= MEAN_TIGHT


def test_full_size_c5_fp64_path_and_oracle_rows(ctx):
    """C5 at full size (4e7 x 768, K=4096; 2.5e14 flops, beyond a CPU run): the fast path
    (tcgen05 nomination + fp64 exact pass) against FSIL_PATH_FP64 (every row refined over
    all K clusters in fp64 with the reference formula and tie rule) on ALL rows, and both
    against the oracle on 3000 sampled rows scored with the oracle's own global aggregates."""
    fast = _full_size_gpu(ctx, "C5")
    full = _full_size_gpu(ctx, "C5", path=PATHS["fp64"], data=(fast["X"], fast["L"], "cosine"))
    mism = np.flatnonzero(fast["nb"] != full["nb"])
    assert mism.size == 0, f"C5: {mism.size} neighbour mismatches vs the fp64 path, rows {mism[:5]}"
    assert np.abs(fast["s"] - full["s"]).max() <= S_TIGHT
    assert abs(fast["mean"] - full["mean"]) <= MEAN_TIGHT
    Xd = fast["X"]
    L = fast["L"].cpu().numpy()
    n = L.shape[0]
    dense, raw = oracle.first_appearance(L)
    assert raw.tolist() == fast["d2r"].tolist() and np.array_equal(dense, fast["own"])
    del fast["X"], full["X"], fast["L"], full["L"]
    X = Xd.cpu().numpy()
    del Xd
    counts, sums, psi = oracle.aggregate_dense(X, dense, fast["k"], "cosine")
    rows = np.random.default_rng(5).choice(n, 3000, replace=False)
    _, _, sv, nbv = oracle.score_rows(X, dense, counts, sums, psi, rows, "cosine", threads=0)
    assert np.array_equal(nbv, fast["nb"][rows])
    assert np.abs(sv - fast["s"][rows]).max() <= S_TIGHT
    print(f"C5 full size: S_fast={fast['mean']:.15f} S_fp64={full['mean']:.15f} "
          f"|dS|={abs(fast['mean'] - full['mean']):.3e}")


def _shard_loopback(X, L, metric, nshards, path=0, device_exchange=False, ctxs=None, attempts=None):
    """The multi-GPU protocol (fsil_shard_*) with `nshards` contexts on one device and
    the three exchanges done in-process (device sums / minima), one shard after the
    other -- the device entry points and the exchange layouts under test, not NCCL.
    `ctxs` reuses contexts across calls (K speculation); a finish that returns FSIL_AGAIN
    on every shard repeats the protocol, as run_sharded does; `attempts` collects how many
    rounds each call took."""
    import torch
    from paper_2303_14102_b200 import Context, ValidationError, plan_shards
    from paper_2303_14102_b200.api import ShardAgain
    from paper_2303_14102_b200.distributed import device_view

    n, d = X.shape
    ranges = plan_shards(n, nshards)
    own = ctxs is None
    if own:
        ctxs = [Context(0) for _ in ranges]
    assert len(ctxs) == len(ranges)
    dev = torch.device("cuda", 0)
    Xd = [torch.from_numpy(X[b:e]).to(dev) for b, e in ranges]
    Ld = [torch.from_numpy(np.asarray(L[b:e], np.int32)).to(dev) for b, e in ranges]
    sd = [torch.empty(e - b, dtype=torch.float64, device=dev) for b, e in ranges]
    nbd = [torch.empty(e - b, dtype=torch.int32, device=dev) for b, e in ranges]

    def one_round():
        if device_exchange:  # buffers gathered in rank order, merged on the device
            bufs = []
            for c, x, l, (b, e) in zip(ctxs, Xd, Ld, ranges):
                c.set_path(path)
                c.set_stream(torch.cuda.current_stream(dev).cuda_stream)
                ptr, cap = c.shard_begin_device(metric, x.data_ptr(), l.data_ptr(), e - b, d, b, n,
                                                f64=x.dtype == torch.float64)
                bufs.append(device_view(ptr, 2 * cap, torch.int64, dev).clone())
            gathered = torch.cat(bufs)
            again = 0
            for c in ctxs:
                try:
                    c.shard_set_dictionary_device(gathered.data_ptr(), len(ctxs), cap)
                except ShardAgain:  # a dictionary outgrew the exchange buffer
                    again += 1
            assert again in (0, len(ctxs)), "FSIL_AGAIN must be seen by every shard alike"
            if again:
                return None
            raw = np.array([], np.int32)
        else:
            first = {}
            for c, x, l, (b, e) in zip(ctxs, Xd, Ld, ranges):
                c.set_path(path)
                c.set_stream(torch.cuda.current_stream(dev).cuda_stream)  # ordered with the exchanges
                nd = c.shard_begin(metric, x.data_ptr(), l.data_ptr(), e - b, d, b, n, f64=x.dtype == torch.float64)
                labs, rows = c.shard_get_dictionary(nd)
                for lab, row in zip(labs.tolist(), rows.tolist()):
                    first[lab] = min(row, first.get(lab, row))
            raw = np.array([lab for lab, _ in sorted(first.items(), key=lambda kv: kv[1])], np.int32)
            for c in ctxs:
                c.shard_set_dictionary(raw)
        stats, checks = [], []
        for c in ctxs:
            ps, ln, pc = c.shard_aggregate()
            stats.append(device_view(ps, ln, torch.float64, dev))
            checks.append(device_view(pc, 2, torch.int64, dev))
        tot = torch.stack(stats).sum(0)
        low = torch.stack(checks).min(0).values
        for st, ch in zip(stats, checks):
            st.copy_(tot)
            ch.copy_(low)
        parts = []
        for c, s_, nb_ in zip(ctxs, sd, nbd):
            parts.append(device_view(c.shard_score(s=s_, neighbour=nb_), 2, torch.float64, dev))
        ptot = torch.stack(parts).sum(0)
        for pp in parts:
            pp.copy_(ptot)
        torch.cuda.synchronize()
        means, errors, again = [], [], 0
        for c in ctxs:
            try:
                means.append(c.shard_finish())
            except ValidationError as e:
                errors.append(str(e))
            except ShardAgain:
                again += 1
        assert again in (0, len(ctxs)), "FSIL_AGAIN must be seen by every shard alike"
        return (means, errors, raw) if again == 0 else None

    try:
        for k in range(1, 9):
            r = one_round()
            if r is not None:
                break
        assert r is not None, "K speculation missed repeatedly"
        if attempts is not None:
            attempts.append(k)
        means, errors, raw = r
        s = torch.cat(sd).cpu().numpy()
        nb = torch.cat(nbd).cpu().numpy()
        return means, errors, s, nb, raw
    finally:
        if own:
            for c in ctxs:
                c.close()


@pytest.mark.parametrize("nshards,metric,path", [(2, "sqeuclid", 0), (3, "cosine", 0), (2, "cosine", 2),
                                                   (4, "sqeuclid", 1)])
def test_shard_protocol_on_device(nshards, metric, path):
    rng = np.random.default_rng(nshards * 7 + path)
    n, d = 20_000, 64
    X = (rng.normal(size=(n, d)) + 3 * rng.normal(size=(12, d))[rng.integers(0, 12, n)]).astype(np.float32)
    L = rng.integers(0, 12, n) * 5 - 17
    L[n - 3:] = 999  # a cluster only the last shard holds
    ref = oracle.silhouette(X, L, metric)
    means, errors, s, nb, raw = _shard_loopback(X, L, metric, nshards, path)
    assert not errors
    assert raw.tolist() == ref.dense_to_raw.tolist()
    for m in means:
        assert abs(m - ref.mean) <= MEAN_TOL
    assert np.abs(s - ref.s).max() <= S_TOL
    assert np.array_equal(nb, ref.neighbour)


def test_shard_protocol_validation_is_global():
    rng = np.random.default_rng(3)
    n, d = 3000, 16
    X = rng.normal(size=(n, d)).astype(np.float32)
    L = rng.integers(0, 5, n)
    X[2500, 3] = np.nan   # last shard
    X[1200, 7] = np.inf   # middle shard: first offender in dataset order
    means, errors, *_ = _shard_loopback(X, L, "sqeuclid", 3)
    assert not means and len(errors) == 3
    assert all(e == "non-finite feature value at point 1200, dimension 7" for e in errors)


@pytest.mark.parametrize("metric", ["sqeuclid", "cosine"])
@pytest.mark.parametrize("offset", [0.0, 1000.0])
def test_fp64_front_end_matches_fp64_oracle(ctx, metric, offset):
    """fsil_silhouette_f64 on features fp32 cannot represent (and, with the offset, whose
    fp32 rounding is far coarser than the cluster spread): aggregation and refinement
    read the fp64 values, so the result is the fp64 reference's -- not the fp32 data's."""
    rng = np.random.default_rng(11 if offset else 12)
    n, d, k = 20_000, 64, 12
    centres = rng.normal(size=(k, d)) * 2.0
    L = rng.integers(0, k, n)
    X = (offset + centres[L] + rng.normal(size=(n, d)) * 0.7).astype(np.float64)
    L = L * 3 + 5
    ref = oracle.silhouette(X, L, metric)
    for path in ("auto", "tcgen05", "fp64"):
        ctx.set_path(PATHS[path])
        got = ctx.silhouette(X, L, metric)
        tag = f"fp64 {metric} offset={offset} path={path}"
        mism = np.flatnonzero(got.neighbour != ref.neighbour)
        if mism.size:
            assert reference_noise_ties(X, ref, metric, mism, got.neighbour[mism]).all(), tag
        assert np.abs(got.s - ref.s).max() <= S_TOL, tag
        assert abs(got.mean - ref.mean) <= MEAN_TOL, tag
    ctx.set_path(0)


def test_fp64_front_end_rejects_ffma(ctx):
    from paper_2303_14102_b200 import FsilError
    X = np.random.default_rng(1).normal(size=(500, 16))
    L = np.arange(500) % 4
    ctx.set_path(PATHS["ffma"])
    try:
        with pytest.raises((ValueError, FsilError)):
            ctx.silhouette(X, L, "sqeuclid")
    finally:
        ctx.set_path(0)


def test_fp64_front_end_sharded():
    rng = np.random.default_rng(5)
    n, d = 9000, 32
    X = (rng.normal(size=(n, d)) * 3 + 50.0).astype(np.float64)
    L = rng.integers(0, 7, n) * 2 + 1
    ref = oracle.silhouette(X, L, "sqeuclid")
    means, errors, s, nb, raw = _shard_loopback(X, L, "sqeuclid", 3, 0)
    assert not errors and raw.tolist() == ref.dense_to_raw.tolist()
    assert all(abs(m - ref.mean) <= MEAN_TOL for m in means)
    assert np.abs(s - ref.s).max() <= S_TOL


@pytest.mark.parametrize("metric", ["sqeuclid", "cosine", "euclid"])
def test_naive_engine_matches_naive_oracle(ctx, metric):
    """fsil_silhouette_naive (every pairwise distance in fp64, naive.cpp:30-71) against the
    oracle's own naive engine -- including plain Euclidean, which only this engine serves."""
    rng = np.random.default_rng(21)
    n, d = 3000, 16
    X = rng.normal(size=(n, d)) + rng.normal(size=(6, d))[rng.integers(0, 6, n)] * 3
    L = rng.integers(0, 6, n) * 7 + 2
    L[17] = 999  # a singleton
    ref = oracle.silhouette(X, L, metric, engine="naive")
    got = ctx.silhouette_naive(X, L, metric)
    assert got.engine == "naive"
    assert np.array_equal(got.neighbour, ref.neighbour)
    assert np.abs(got.s - ref.s).max() <= 1e-12
    assert np.allclose(got.a, ref.a, rtol=1e-12, atol=1e-12) and np.allclose(got.b, ref.b, rtol=1e-12, atol=1e-12)
    assert abs(got.mean - ref.mean) <= 1e-13


def test_compare_fast_against_naive():
    """The reference's compare contract (tools/main.cpp:62-108) on the GPU engines."""
    from paper_2303_14102_b200.api import compare
    rng = np.random.default_rng(22)
    X = rng.normal(size=(4000, 32)) + rng.normal(size=(5, 32))[rng.integers(0, 5, 4000)] * 2
    L = rng.integers(0, 5, 4000)
    # the fast engine's contract: |ds_i| <= 1e-5 (absolute), a_i/b_i to ~1e-5 relative
    for metric in ("cosine", "sqeuclid"):
        ok = compare(X, L, metric, rtol=1e-4, atol=S_TOL)
        assert ok["within"] and abs(ok["fast_mean"] - ok["naive_mean"]) <= MEAN_TOL, (metric, ok)
    bad = compare(X, L, "cosine", rtol=1e-4, atol=S_TOL, inject_fault=1e-3)
    assert not bad["within"] and bad["max_abs_deviation"] >= 1e-3 * 0.99


def test_cli_score_and_compare(tmp_path):
    """The reference tool's score / compare over the GPU engines: CSV in, report out,
    exit codes 0 (ok) and 3 (tolerance exceeded) -- tools/main.cpp:19-108."""
    import json
    import subprocess
    import sys
    from paper_2303_14102_b200.io import CsvDataset, write_points_csv
    rng = np.random.default_rng(31)
    X = rng.normal(size=(1500, 8)) + rng.normal(size=(4, 8))[rng.integers(0, 4, 1500)] * 3
    L = rng.integers(0, 4, 1500).astype(np.int32)
    csv = tmp_path / "pts.csv"
    write_points_csv(CsvDataset(X, L, ["w", "x", "y", "z"]), csv)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2303_14102_b200", *a], cwd=root,
                                    capture_output=True, text=True, timeout=300)
    out = tmp_path / "rep.jsonl"
    r = run("score", "--input", str(csv), "--metric", "cosine", "--output", str(out))
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in out.read_text().splitlines()]
    ref = oracle.silhouette(X, L, "cosine")
    assert len(lines) == 1501 and abs(lines[-1]["mean"] - ref.mean) <= MEAN_TOL
    assert max(abs(p["s"] - ref.s[p["index"]]) for p in lines[:-1]) <= S_TOL
    assert run("score", "--input", str(csv), "--engine", "naive", "--format", "csv").returncode == 0
    assert run("compare", "--input", str(csv)).returncode == 0
    assert run("compare", "--input", str(csv), "--inject-fault", "1e-3").returncode == 3


@pytest.mark.parametrize("nshards,metric,path", [(2, "sqeuclid", 0), (3, "cosine", 2), (4, "cosine", 0)])
def test_shard_protocol_device_exchange(nshards, metric, path):
    """The dictionary exchanged and merged on the device (what bench.py --gpus N uses):
    same global first-appearance order and results as one process."""
    rng = np.random.default_rng(nshards * 13 + path)
    n, d = 20_000, 64
    X = (rng.normal(size=(n, d)) + 3 * rng.normal(size=(12, d))[rng.integers(0, 12, n)]).astype(np.float32)
    L = rng.integers(0, 12, n) * 5 - 17
    L[n - 3:] = 999  # a cluster only the last shard holds
    L[:2] = 4242     # and one that the first shard holds first
    ref = oracle.silhouette(X, L, metric)
    means, errors, s, nb, _ = _shard_loopback(X, L, metric, nshards, path, device_exchange=True)
    assert not errors
    for m in means:
        assert abs(m - ref.mean) <= MEAN_TOL
    assert np.abs(s - ref.s).max() <= S_TOL
    assert np.array_equal(nb, ref.neighbour)


def test_k_speculation_sequence():
    """One context, K changing from call to call: each call's kernels are launched for the
    previous call's K and checked at the end (a miss repeats the call unspeculated).  Hits,
    misses up and down, the multi-block ordering in both directions and K = 1 all give the
    oracle's answer."""
    from paper_2303_14102_b200 import Context, ValidationError
    c = Context(0)
    try:
        rng = np.random.default_rng(21)
        for n, d, k in [(4000, 16, 6), (4000, 16, 6), (5000, 24, 9), (3000, 8, 3), (3000, 8, 3),
                        (6000, 12, 3000), (6000, 12, 3000), (2000, 12, 40), (2000, 8, 2)]:
            X = (rng.normal(size=(n, d)) + rng.normal(size=(1, d)) * 2).astype(np.float32)
            L = rng.permutation(np.arange(n) % k) * 3 + 1
            for metric in ("sqeuclid", "cosine"):
                check(c, X, L, metric, label=f"spec k={k}")
        X = rng.normal(size=(500, 4)).astype(np.float32)
        with pytest.raises(ValidationError, match="single cluster"):
            c.silhouette(X, np.full(500, 7), "sqeuclid")
        check(c, X, np.arange(500) % 5, "sqeuclid", label="after K=1")
    finally:
        c.close()


def test_shard_k_speculation_again():
    """Sharded device exchange with contexts reused: the first call waits for the count,
    a call with a new K misses on every shard alike (FSIL_AGAIN) and is repeated, a call
    with the same K is served by the speculation."""
    from paper_2303_14102_b200 import Context
    ctxs = [Context(0) for _ in range(3)]
    try:
        rng = np.random.default_rng(5)
        n, d = 9000, 32
        attempts = []
        for k in (7, 11, 11, 4):
            X = (rng.normal(size=(n, d)) + 2 * rng.normal(size=(k, d))[rng.integers(0, k, n)]).astype(np.float32)
            L = rng.permutation(np.arange(n) % k) * 5 - 2
            ref = oracle.silhouette(X, L, "cosine")
            means, errors, s, nb, _ = _shard_loopback(X, L, "cosine", 3, 0, device_exchange=True, ctxs=ctxs,
                                                      attempts=attempts)
            assert not errors
            assert all(abs(m - ref.mean) <= MEAN_TOL for m in means)
            assert np.abs(s - ref.s).max() <= S_TOL and np.array_equal(nb, ref.neighbour)
        assert attempts == [1, 2, 1, 2], attempts
    finally:
        for c in ctxs:
            c.close()


def test_shard_exchange_overflow_again():
    """More distinct labels per rank than the device exchange holds (its first capacity
    is 63 entries): every shard returns FSIL_AGAIN, the repeat uses a larger buffer;
    also when the overflow is only seen at finish (speculated call), and across the
    multi-block ordering (K > 2048)."""
    from paper_2303_14102_b200 import Context
    ctxs = [Context(0) for _ in range(3)]
    try:
        rng = np.random.default_rng(9)
        n, d = 12_000, 16
        attempts = []
        for k in (500, 500, 3000, 3000):
            X = (rng.normal(size=(n, d)) + 2 * rng.normal(size=(k, d))[rng.integers(0, k, n)]).astype(np.float32)
            L = rng.permutation(np.arange(n) % k) * 3 + 11
            ref = oracle.silhouette(X, L, "sqeuclid")
            means, errors, s, nb, _ = _shard_loopback(X, L, "sqeuclid", 3, 0, device_exchange=True, ctxs=ctxs,
                                                      attempts=attempts)
            assert not errors
            assert all(abs(m - ref.mean) <= MEAN_TOL for m in means)
            assert np.abs(s - ref.s).max() <= S_TOL and np.array_equal(nb, ref.neighbour)
        assert attempts == [2, 1, 2, 1], attempts
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("name,n,nshards", [("C2", 200_000, 2), ("C3", 400_000, 4), ("C4", 300_000, 8),
                                            ("C5", 60_000, 3)])
def test_strong_scaling_shards_match_single_gpu(ctx, name, n, nshards):
    """bench.py's strong scaling: each rank generates its plan_shards rows of ONE global
    dataset (datagen rows=...), byte-identical to those rows of the whole, and the sharded
    protocol over those shards reproduces the single-GPU result: S within 1e-12 (only the
    order of the all-reduced fp64 sums differs), neighbours identical, s_i within 1e-12."""
    import torch
    from paper_2303_14102_b200 import datagen, plan_shards
    Xw, Lw, metric = datagen.generate_device(name, n=n)
    for b, e in plan_shards(n, nshards):
        Xs, Ls, _ = datagen.generate_device(name, n=n, rows=(b, e))
        assert torch.equal(Xs, Xw[b:e]) and torch.equal(Ls, Lw[b:e]), (b, e)
    X, L = Xw.cpu().numpy(), Lw.cpu().numpy()
    del Xw, Lw
    single = ctx.silhouette(X, L, metric)
    means, errors, s, nb, _ = _shard_loopback(X, L, metric, nshards, device_exchange=True)
    assert not errors and all(abs(m - single.mean) <= 1e-12 for m in means), (means, single.mean)
    assert np.array_equal(nb, single.neighbour)
    assert np.abs(s - single.s).max() <= 1e-12
