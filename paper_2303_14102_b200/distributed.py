"""Multi-GPU row sharding: one process per GPU, torch.distributed (NCCL) for the
three exchange steps of the sharded protocol in include/fsil.h.

Reference behaviour mirrored: the reference's only parallelism is data
parallelism over contiguous row ranges (plan_shards, engine.cpp:8-25) with
block partials "collected on a node" and folded (engine.hpp:75-78, PAPER.md
section 3 footnotes) and the merged statistics broadcast to every scoring
shard (engine.hpp:93-101).  Here:

  exchange 1  first-appearance dictionary: all-gather of each rank's
              (raw label, first global row) pairs, merged by minimum first row
              and ordered by it, so every rank derives the same dense ids
              (dataset.cpp:41-51 over the whole dataset);
  exchange 2  all-reduce SUM of the K*(D+2) (or K*(D+1)) fp64 cluster
              statistics, all-reduce MIN of the int64 validation word;
  exchange 3  all-reduce SUM of (sum of s_i, refined-row count).

No per-point data crosses ranks.  The exchange logic is written against a small
`ShardOps` interface so it is testable on CPU with the gloo backend; the
production ops are `CudaShardOps` over libfsil.
"""
from __future__ import annotations

from typing import Optional, Protocol, Tuple

import numpy as np
import torch
import torch.distributed as dist


class ShardOps(Protocol):
    def begin(self) -> Tuple[np.ndarray, np.ndarray]: ...          # local (labels, first rows)
    def set_dictionary(self, raw_in_dense_order: np.ndarray) -> None: ...
    def aggregate(self) -> Tuple[torch.Tensor, torch.Tensor]: ...  # (stats f64, checks i64[2])
    def score(self) -> torch.Tensor: ...                           # f64[2]
    def finish(self) -> float: ...


def merge_dictionaries(labels: np.ndarray, first_rows: np.ndarray, device, group=None) -> np.ndarray:
    """All-gather every rank's distinct labels with their first global row; return the
    global raw labels ordered by first appearance (identical on every rank)."""
    world = dist.get_world_size(group)
    n_local = torch.tensor([labels.shape[0]], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(counts, n_local, group=group)
    width = int(max(int(c.item()) for c in counts))
    pad = torch.full((2, max(width, 1)), -1, dtype=torch.int64, device=device)
    if labels.shape[0]:
        pad[0, : labels.shape[0]] = torch.from_numpy(labels.astype(np.int64)).to(device)
        pad[1, : labels.shape[0]] = torch.from_numpy(first_rows.astype(np.int64)).to(device)
    gathered = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(gathered, pad, group=group)
    first = {}
    for r, g in enumerate(gathered):
        g = g.cpu().numpy()
        for lab, row in zip(g[0, : int(counts[r].item())], g[1, : int(counts[r].item())]):
            lab, row = int(lab), int(row)
            if lab not in first or row < first[lab]:
                first[lab] = row
    order = sorted(first.items(), key=lambda kv: kv[1])
    return np.array([lab for lab, _ in order], dtype=np.int32)


def run_sharded(ops: ShardOps, device, group=None) -> float:
    """The three-exchange protocol; returns the global mean silhouette S.  Ops with a
    device dictionary exchange (CudaShardOps) gather and merge the dictionaries on the
    GPUs; others go through the host merge."""
    from .api import ShardAgain
    for _ in range(8):
        try:
            return _sharded_round(ops, device, group)
        except ShardAgain:
            # every rank alike: the speculated K missed (raised by finish) or a dictionary
            # outgrew the device exchange (raised by the dictionary step): repeat
            continue
    raise RuntimeError("sharded protocol: repeated FSIL_AGAIN")


def _sharded_round(ops: ShardOps, device, group=None) -> float:
    if hasattr(ops, "exchange_dictionary"):
        ops.exchange_dictionary(group)
    else:
        labels, rows = ops.begin()
        raw = merge_dictionaries(labels, rows, device, group)
        ops.set_dictionary(raw)
    stats, checks = ops.aggregate()
    dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    # the validation word is only read by finish: its MIN overlaps the scoring kernels
    pending = dist.all_reduce(checks, op=dist.ReduceOp.MIN, group=group, async_op=True)
    partial = ops.score()
    dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    pending.wait()
    return ops.finish()


class _DeviceArray:
    """Zero-copy view of a libfsil device buffer for torch (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


_VIEWS = {}


def device_view(ptr: int, n: int, dtype: torch.dtype, device) -> torch.Tensor:
    """A non-owning tensor over n elements at ptr.  Cached by (ptr, n, dtype): libfsil's
    buffers are stable from call to call, and building the view is host time on every
    step of the protocol."""
    key = (ptr, n, dtype, str(device))
    v = _VIEWS.get(key)
    if v is None:
        if len(_VIEWS) >= 256:
            _VIEWS.clear()
        typestr = {torch.float64: "<f8", torch.int64: "<i8"}[dtype]
        v = _VIEWS[key] = torch.as_tensor(_DeviceArray(ptr, n, typestr), device=device)
    return v


_GATHER = {}


def _gather_buffer(n: int, device) -> torch.Tensor:
    key = (n, str(device))
    buf = _GATHER.get(key)
    if buf is None:
        _GATHER.clear()
        buf = _GATHER[key] = torch.empty(n, dtype=torch.int64, device=device)
    return buf


class CudaShardOps:
    """Production ops: libfsil kernels on this rank's resident rows."""

    def __init__(self, ctx, metric, X: torch.Tensor, labels: torch.Tensor, row_offset: int,
                 n_global: int, s: Optional[torch.Tensor] = None,
                 neighbour: Optional[torch.Tensor] = None):
        self.ctx, self.metric, self.X, self.L = ctx, metric, X, labels
        self.row_offset, self.n_global = row_offset, n_global
        self.s, self.nb = s, neighbour
        self.device = X.device
        # kernels run on torch's current stream, so NCCL orders after them
        ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def exchange_dictionary(self, group=None):
        """Device exchange: local (label, first row) pairs -> all-gather (NCCL) -> merged
        on every GPU (fsil_shard_begin_device / fsil_shard_set_dictionary_device)."""
        n, d = self.X.shape
        ptr, cap = self.ctx.shard_begin_device(self.metric, self.X.data_ptr(), self.L.data_ptr(), n, d,
                                               self.row_offset, self.n_global, f64=self.X.dtype == torch.float64)
        local = device_view(ptr, 2 * cap, torch.int64, self.device)
        world = dist.get_world_size(group)
        gathered = _gather_buffer(world * 2 * cap, self.device)
        dist.all_gather_into_tensor(gathered, local, group=group)
        self.ctx.shard_set_dictionary_device(gathered.data_ptr(), world, cap)

    def begin(self):
        n, d = self.X.shape
        nd = self.ctx.shard_begin(self.metric, self.X.data_ptr(), self.L.data_ptr(), n, d,
                                  self.row_offset, self.n_global, f64=self.X.dtype == torch.float64)
        return self.ctx.shard_get_dictionary(nd)

    def set_dictionary(self, raw):
        self.ctx.shard_set_dictionary(raw)

    def aggregate(self):
        ps, ln, pc = self.ctx.shard_aggregate()
        return (device_view(ps, ln, torch.float64, self.device),
                device_view(pc, 2, torch.int64, self.device))

    def score(self):
        pp = self.ctx.shard_score(s=self.s, neighbour=self.nb)
        return device_view(pp, 2, torch.float64, self.device)

    def finish(self):
        return self.ctx.shard_finish()


def compute_silhouette_sharded(ctx, metric, X: torch.Tensor, labels: torch.Tensor,
                               row_offset: int, n_global: int, s=None, neighbour=None,
                               group=None) -> float:
    """This rank's rows [row_offset, row_offset + len(X)) of an n_global-row dataset;
    per-point outputs stay on this rank's GPU; returns the global mean S."""
    ops = CudaShardOps(ctx, metric, X, labels, row_offset, n_global, s, neighbour)
    return run_sharded(ops, X.device, group)
