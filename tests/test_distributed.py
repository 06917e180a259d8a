"""Multi-rank exchange logic (paper_2303_14102_b200.distributed) on CPU with the
gloo backend, world_size 2 and 3.  The per-rank device phases are stood in for by
test-only CPU ops over the oracle (the checker); what is under test is the
product's protocol: first-appearance dictionary merge across shards, the
statistics all-reduce layout, the validation-word MIN and the final mean."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2303_14102_b200.distributed import merge_dictionaries, run_sharded


class OracleShardOps:
    """CPU stand-in for CudaShardOps: same buffers and layouts (include/fsil.h)."""

    def __init__(self, metric, X, L, row_offset):
        self.metric, self.X, self.L, self.off = metric, X, L, row_offset

    def begin(self):
        uniq, first = np.unique(self.L, return_index=True)
        order = np.argsort(first)
        return uniq[order].astype(np.int32), (first[order] + self.off).astype(np.int64)

    def set_dictionary(self, raw):
        self.raw = raw
        pos = {int(v): i for i, v in enumerate(raw)}
        self.dense = np.array([pos[int(v)] for v in self.L], np.int32)

    def aggregate(self):
        k, d = len(self.raw), self.X.shape[1]
        cos = self.metric == "cosine"
        counts = np.bincount(self.dense, minlength=k).astype(np.float64)
        X64 = self.X.astype(np.float64)
        if cos:
            X64 = X64 / np.linalg.norm(X64, axis=1, keepdims=True)
        sums = np.zeros((k, d))
        np.add.at(sums, self.dense, X64)
        parts = [counts] + ([] if cos else [np.bincount(self.dense, (self.X.astype(np.float64) ** 2).sum(1), k)])
        self.stats = torch.from_numpy(np.concatenate(parts + [sums.ravel()]))
        bad = np.argwhere(~np.isfinite(self.X))
        first_bad = (self.off + bad[0][0]) * d + bad[0][1] if len(bad) else np.iinfo(np.int64).max
        self.checks = torch.tensor([first_bad, np.iinfo(np.int64).max], dtype=torch.int64)
        return self.stats, self.checks

    def score(self):
        k, d = len(self.raw), self.X.shape[1]
        st = self.stats.numpy()
        counts = st[:k].astype(np.int64)
        psi = None if self.metric == "cosine" else st[k:2 * k]
        sums = st[(k if self.metric == "cosine" else 2 * k):].reshape(k, d)
        _, _, s, _ = oracle.score_rows(self.X, self.dense, counts, sums, psi,
                                       np.arange(self.X.shape[0]), self.metric)
        self.part = torch.tensor([s.sum(), 0.0], dtype=torch.float64)
        return self.part

    def finish(self):
        # same decoding of the MIN-reduced validation word as fsil_shard_finish (capi.cu)
        bad = int(self.checks[0])
        if bad != np.iinfo(np.int64).max:
            d = self.X.shape[1]
            raise ValueError(f"non-finite feature value at point {bad // d}, dimension {bad % d}")
        return float(self.part[0]) / self.n_global


def _worker(rank, world, port, metric, X, L, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = X.shape[0]
    ranges = oracle.plan_shards(n, world)
    b, e = ranges[rank]
    ops = OracleShardOps(metric, X[b:e], L[b:e], b)
    ops.n_global = n
    try:
        mean = run_sharded(ops, torch.device("cpu"))
        ret[rank] = (mean, ops.raw.tolist())
    except ValueError as e:
        ret[rank] = ("error", str(e))
    dist.destroy_process_group()


def _run(world, metric, X, L, port):
    ret = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, metric, X, L, ret), nprocs=world, join=True)
    return [ret[r] for r in range(world)]


@pytest.mark.parametrize("world,metric", [(2, "sqeuclid"), (2, "cosine"), (3, "sqeuclid")])
def test_sharded_protocol_matches_single_process(world, metric):
    rng = np.random.default_rng(world * 10 + len(metric))
    n = 1201
    X = (rng.normal(size=(n, 6)) + rng.normal(size=(1, 6)) * 2).astype(np.float32)
    # labels whose first appearances straddle the shard boundary, out of numeric order
    L = rng.integers(0, 9, n) * 13 - 40
    L[n - 5:] = 777  # a cluster that only the last shard sees
    ref = oracle.silhouette(X, L, metric)
    out = _run(world, metric, X, L, 29500 + world * 7 + len(metric))
    for mean, raw in out:
        assert raw == ref.dense_to_raw.tolist(), "dense order must be global first appearance"
        assert abs(mean - ref.mean) <= 1e-12


def test_merge_dictionaries_single_rank():
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        raw = merge_dictionaries(np.array([9, 4, 2], np.int32), np.array([5, 0, 3]), torch.device("cpu"))
        assert raw.tolist() == [4, 2, 9]
    finally:
        dist.destroy_process_group()


def test_sharded_validation_error_is_global():
    """A non-finite value on any shard fails every rank with the same message, naming
    the lowest global (row, dimension) -- the reference's first-offender order
    (dataset.cpp:35-37) -- via the MIN all-reduce of the validation word."""
    rng = np.random.default_rng(7)
    n, d, world = 900, 5, 3
    X = rng.normal(size=(n, d)).astype(np.float32)
    L = rng.integers(0, 4, n)
    X[700, 2] = np.nan   # shard 2
    X[450, 4] = np.inf   # shard 1: the first offender in dataset order
    out = _run(world, "sqeuclid", X, L, 29587)
    for tag, msg in out:
        assert tag == "error"
        assert msg == "non-finite feature value at point 450, dimension 4"
