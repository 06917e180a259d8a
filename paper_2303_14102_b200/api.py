"""Python host mirror of the reference's entry points over the C ABI (libfsil.so).

Reference interface mirrored (names, argument meaning, error behaviour):
  compute_silhouette(ds, metric, engine, shards)   engine.hpp:124-125, engine.cpp:76-92
  validate_and_densify(points, labels)             dataset.hpp:46, dataset.cpp:26-68 (fused)
  plan_shards(n, w)                                engine.cpp:8-25
  assemble_score(a, b)                             report.cpp:7-14
  PointScore / SilhouetteReport                    report.hpp:10-26
  ValidationError / IoError                        types.hpp:41-50

The compute path is libfsil.so (hand-written sm_100a kernels); there is no CPU
fallback: without the built library or a B200 every call raises.
"""
from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSIL_LIB_PATH") or os.path.join(_PKG, "libfsil.so")  # override: A/B builds
DATAGEN_PATH = os.path.join(_PKG, "libfsil_datagen.so")

SQEUCLID, COSINE, EUCLID = 0, 1, 2
PATH_AUTO, PATH_FFMA, PATH_TCGEN05, PATH_FP64 = 0, 1, 2, 3
_METRIC_TAGS = {SQEUCLID: "squared_euclidean", COSINE: "cosine", EUCLID: "euclidean_oracle"}

# FSIL status codes (include/fsil.h)
OK, ERR_IO, ERR_VALIDATION, ERR_INVALID_ARGUMENT, ERR_CUDA, ERR_NCCL, ERR_INTERNAL, AGAIN = range(8)

# fsil.h entry points: name -> (restype, argtypes)
_P = ctypes.c_void_p
_I64, _I32, _DBL = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
EXPORTS = {
    "fsil_abi_version": (ctypes.c_int, []),
    "fsil_create": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int]),
    "fsil_destroy": (None, [_P]),
    "fsil_last_error": (ctypes.c_char_p, [_P]),
    "fsil_set_stream": (ctypes.c_int, [_P, _P]),
    "fsil_set_path": (ctypes.c_int, [_P, ctypes.c_int]),
    "fsil_set_timing": (ctypes.c_int, [_P, ctypes.c_int]),
    "fsil_get_stats": (ctypes.c_int, [_P, _P]),
    "fsil_silhouette": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _I32, _P, _P, _P, _P, _P,
                                       _P, _P, _P]),
    "fsil_silhouette_device": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _I32, _P, _P, _P,
                                              _P, _P, _P, _P, _P]),
    "fsil_silhouette_f64": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _I32, _P, _P, _P, _P, _P,
                                           _P, _P, _P]),
    "fsil_silhouette_device_f64": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _I32, _P, _P, _P,
                                                  _P, _P, _P, _P, _P]),
    "fsil_silhouette_naive": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _I32, _P, _P, _P, _P,
                                             _P, _P, _P, _P]),
    "fsil_shard_begin": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _I32, _I64, _I64, _P]),
    "fsil_shard_begin_f64": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _I32, _I64, _I64, _P]),
    "fsil_shard_begin_device": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int, _P, _I64, _I32, _I64, _I64,
                                               _P, _P]),
    "fsil_shard_set_dictionary_device": (ctypes.c_int, [_P, _P, _I32, _I64]),
    "fsil_shard_get_dictionary": (ctypes.c_int, [_P, _P, _P]),
    "fsil_shard_set_dictionary": (ctypes.c_int, [_P, _P, _I32]),
    "fsil_shard_aggregate": (ctypes.c_int, [_P, _P, _P, _P]),
    "fsil_shard_score": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "fsil_shard_finish": (ctypes.c_int, [_P, _P]),
    "fsil_plan_shards": (ctypes.c_int, [_I64, _I32, _P, _P]),
    "fsil_assemble_score": (ctypes.c_int, [_DBL, _DBL, _P]),
}


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the (synchronising) legacy default stream


class ValidationError(ValueError):
    """fastsil::ValidationError (types.hpp:41-44): a dataset/argument invariant."""


class IoError(OSError):
    """fastsil::IoError (types.hpp:47-50)."""


class FsilError(RuntimeError):
    """CUDA / collective / internal failure reported by libfsil."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[fsil status {status}] {msg}")
        self.status = status


class ShardAgain(FsilError):
    """FSIL_AGAIN from fsil_shard_finish: the speculated global K missed (every rank sees
    it); the protocol is repeated from fsil_shard_begin_device."""


class fsil_stats(ctypes.Structure):
    _fields_ = [("n", _I64), ("d", _I32), ("k", _I32), ("path", _I32), ("agg_path", _I32),
                ("flagged_rows", _I64), ("exact_rows", _I64), ("kernel_launches", _I64), ("ms_densify", ctypes.c_float),
                ("ms_aggregate", ctypes.c_float), ("ms_score", ctypes.c_float),
                ("ms_refine", ctypes.c_float), ("ms_finalize", ctypes.c_float),
                ("ms_score_kernel", ctypes.c_float), ("pair_rows", _I64), ("tc_mmas", _I32), ("tc_threshold", _I32),
                ("rescored_rows", _I64)]


_lib = None


def lib():
    """Load libfsil.so (built in-tree by __graft_entry__.build()).  Fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FsilError(ERR_INTERNAL, f"{LIB_PATH} is not built; run "
                            "`python -m paper_2303_14102_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _raise(status: int, msg: str):
    if status == ERR_VALIDATION:
        raise ValidationError(msg)
    if status == ERR_IO:
        raise IoError(msg)
    if status == ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == AGAIN:
        raise ShardAgain(status, msg)
    raise FsilError(status, msg)


def metric_code(metric) -> int:
    """parse_metric (types.cpp:21-28): CLI spellings plus report tags."""
    if isinstance(metric, (int, np.integer)):
        return int(metric)
    m = {"sqeuclid": SQEUCLID, "squared_euclidean": SQEUCLID, "cosine": COSINE,
         "euclid": EUCLID, "euclidean": EUCLID, "euclidean_oracle": EUCLID}.get(metric)
    if m is None:
        raise ValidationError(f"unknown metric '{metric}' (use sqeuclid or cosine)")
    return m


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


@dataclass
class SilhouetteReport:
    """SilhouetteReport + PointScore (report.hpp:10-26), struct-of-arrays."""
    s: np.ndarray
    neighbour: np.ndarray
    own: Optional[np.ndarray]
    a: Optional[np.ndarray]
    b: Optional[np.ndarray]
    mean: float
    metric: str
    engine: str = "fast"
    shards: int = 1
    wall_time_ms: float = 0.0
    cluster_names: list = field(default_factory=list)  # dense id -> raw label


class Context:
    """One libfsil context bound to one CUDA device (fsil_create / fsil_destroy)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = ctypes.c_void_p()
        st = L.fsil_create(ctypes.byref(h), device)
        if st != OK:
            _raise(st, L.fsil_last_error(None).decode())
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            lib().fsil_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, st):
        if st != OK:
            _raise(st, lib().fsil_last_error(self._h).decode())

    # -- configuration --------------------------------------------------------
    def set_stream(self, stream_handle: Optional[int]):
        """Run on `stream_handle` (a cudaStream_t as int, e.g. torch's
        `current_stream().cuda_stream`).  0 -- torch's default stream -- means the
        legacy default stream (cudaStreamLegacy), so the kernels order with torch
        and NCCL work on it; None returns to a context-owned stream."""
        if stream_handle == 0:
            stream_handle = CUDA_STREAM_LEGACY
        self._check(lib().fsil_set_stream(self._h, stream_handle))

    def set_path(self, path: int):
        self._check(lib().fsil_set_path(self._h, int(path)))

    def set_timing(self, on: bool):
        self._check(lib().fsil_set_timing(self._h, int(bool(on))))

    def stats(self) -> dict:
        s = fsil_stats()
        self._check(lib().fsil_get_stats(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in fsil_stats._fields_}

    # -- whole dataset ----------------------------------------------------------
    def silhouette_naive(self, X, labels, metric="sqeuclid") -> SilhouetteReport:
        """fsil_silhouette_naive: the Theta(N^2 D) engine (naive.cpp:30-71) on the GPU, every
        pairwise distance in fp64; the only engine for metric "euclid"."""
        return self.silhouette(X, labels, metric, want_ab=True, _naive=True)

    def silhouette(self, X, labels, metric="sqeuclid", want_ab=True, _naive=False) -> SilhouetteReport:
        """fsil_silhouette over host arrays (copies in and out of HBM).  float64 features
        take the fp64 front end (fsil_silhouette_f64: exact aggregation and refinement
        on the caller's values, the reference's own Matrix type); anything else is fp32."""
        m = metric_code(metric)
        f64 = _naive or getattr(X, "dtype", None) == np.float64
        X = np.ascontiguousarray(X, dtype=np.float64 if f64 else np.float32)
        if X.ndim != 2:
            X = X.reshape(X.shape[0], -1)
        n, d = X.shape
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        if labels.shape[0] != n:
            raise ValidationError(f"label count ({labels.shape[0]}) does not match point count ({n})")
        s = np.empty(n, np.float64)
        nb = np.empty(n, np.int32)
        own = np.empty(n, np.int32)
        a = np.empty(n, np.float64) if want_ab else None
        b = np.empty(n, np.float64) if want_ab else None
        mean = ctypes.c_double(0.0)
        k = ctypes.c_int32(0)
        d2r = np.empty(max(n, 1), np.int32)
        t0 = time.perf_counter()
        entry = (lib().fsil_silhouette_naive if _naive else
                 lib().fsil_silhouette_f64 if f64 else lib().fsil_silhouette)
        self._check(entry(self._h, m, _ptr(X), _ptr(labels), n, d, _ptr(s), _ptr(nb), _ptr(own), _ptr(a),
                          _ptr(b), ctypes.byref(mean), ctypes.byref(k), _ptr(d2r)))
        wall = (time.perf_counter() - t0) * 1e3
        return SilhouetteReport(s, nb, own, a, b, mean.value, _METRIC_TAGS[m], "naive" if _naive else "fast",
                                1, wall, d2r[: k.value].tolist())

    def silhouette_device(self, X, labels, metric="sqeuclid", s=None, neighbour=None, own=None,
                          a=None, b=None, dense_to_raw=None):
        """fsil_silhouette_device: X [n,d] fp32 (or fp64: the fp64 front end) and labels
        [n] int32 are CUDA tensors (or raw device pointers via silhouette_device_ptr)."""
        n, d = X.shape
        f64 = str(getattr(X, "dtype", "")) == "torch.float64"
        return self.silhouette_device_ptr(X.data_ptr(), labels.data_ptr(), n, d, metric, s,
                                          neighbour, own, a, b, dense_to_raw, f64=f64)

    def silhouette_device_ptr(self, x_ptr, l_ptr, n, d, metric="sqeuclid", s=None, neighbour=None,
                              own=None, a=None, b=None, dense_to_raw=None, f64=False):
        m = metric_code(metric)
        mean = ctypes.c_double(0.0)
        k = ctypes.c_int32(0)
        entry = lib().fsil_silhouette_device_f64 if f64 else lib().fsil_silhouette_device
        self._check(entry(self._h, m, x_ptr, l_ptr, n, d, _ptr(s), _ptr(neighbour), _ptr(own), _ptr(a),
                          _ptr(b), ctypes.byref(mean), ctypes.byref(k), _ptr(dense_to_raw)))
        return mean.value, k.value

    # -- sharded protocol (see include/fsil.h) ------------------------------------
    def shard_begin(self, metric, x_ptr, l_ptr, n_local, d, row_offset, n_global, f64=False) -> int:
        nd = ctypes.c_int64(0)
        entry = lib().fsil_shard_begin_f64 if f64 else lib().fsil_shard_begin
        self._check(entry(self._h, metric_code(metric), x_ptr, l_ptr, n_local, d, row_offset, n_global,
                          ctypes.byref(nd)))
        return nd.value

    def shard_begin_device(self, metric, x_ptr, l_ptr, n_local, d, row_offset, n_global, f64=False):
        """Device dictionary exchange, pass 1: (entries device pointer, capacity)."""
        ptr, cap = ctypes.c_void_p(), ctypes.c_int64(0)
        self._check(lib().fsil_shard_begin_device(self._h, metric_code(metric), x_ptr, 1 if f64 else 0, l_ptr,
                                                  n_local, d, row_offset, n_global, ctypes.byref(ptr),
                                                  ctypes.byref(cap)))
        return ptr.value, cap.value

    def shard_set_dictionary_device(self, gathered_ptr, nranks, capacity):
        self._check(lib().fsil_shard_set_dictionary_device(self._h, gathered_ptr, nranks, capacity))

    def shard_get_dictionary(self, n_distinct):
        labs = np.empty(max(n_distinct, 1), np.int32)
        rows = np.empty(max(n_distinct, 1), np.int64)
        self._check(lib().fsil_shard_get_dictionary(self._h, _ptr(labs), _ptr(rows)))
        return labs[:n_distinct], rows[:n_distinct]

    def shard_set_dictionary(self, raw_in_dense_order):
        raw = np.ascontiguousarray(raw_in_dense_order, dtype=np.int32)
        self._check(lib().fsil_shard_set_dictionary(self._h, _ptr(raw), raw.shape[0]))

    def shard_aggregate(self):
        ps, ln, pc = ctypes.c_void_p(), ctypes.c_int64(0), ctypes.c_void_p()
        self._check(lib().fsil_shard_aggregate(self._h, ctypes.byref(ps), ctypes.byref(ln),
                                               ctypes.byref(pc)))
        return ps.value, ln.value, pc.value

    def shard_score(self, s=None, neighbour=None, own=None, a=None, b=None):
        pp = ctypes.c_void_p()
        self._check(lib().fsil_shard_score(self._h, _ptr(s), _ptr(neighbour), _ptr(own), _ptr(a),
                                           _ptr(b), ctypes.byref(pp)))
        return pp.value

    def shard_finish(self) -> float:
        mean = ctypes.c_double(0.0)
        self._check(lib().fsil_shard_finish(self._h, ctypes.byref(mean)))
        return mean.value


_default_ctx: Optional[Context] = None


def default_context(device: int = 0) -> Context:
    global _default_ctx
    if _default_ctx is None or _default_ctx.device != device:
        _default_ctx = Context(device)
    return _default_ctx


def compute_silhouette(X, labels, metric="sqeuclid", engine="fast", shards: int = 0,
                       device: int = 0) -> SilhouetteReport:
    """compute_silhouette(validate_and_densify(X, labels), metric, engine, shards)
    (engine.cpp:76-92) on one B200.  `shards` is accepted for signature parity (the
    reference's CPU thread count); the device decomposition is fixed by the kernels.
    Multi-GPU row sharding lives in paper_2303_14102_b200.distributed."""
    if engine not in ("fast", "naive"):
        raise ValidationError(f"unknown engine '{engine}' (use fast or naive)")
    ctx = default_context(device)
    rep = ctx.silhouette_naive(X, labels, metric) if engine == "naive" else ctx.silhouette(X, labels, metric)
    rep.shards = shards if shards > 0 else 1
    return rep


def plan_shards(n: int, w: int):
    """plan_shards (engine.cpp:8-25) -> list of (begin, end)."""
    if n < 1:
        raise ValueError("plan_shards: need at least one point")
    if w < 1:
        raise ValueError("plan_shards: need at least one worker")
    ranges = np.empty(2 * min(w, n), np.int64)
    ns = ctypes.c_int32(0)
    st = lib().fsil_plan_shards(n, w, _ptr(ranges), ctypes.byref(ns))
    if st != OK:
        _raise(st, "plan_shards failed")
    return [(int(ranges[2 * i]), int(ranges[2 * i + 1])) for i in range(ns.value)]


def assemble_score(a: float, b: float) -> float:
    """assemble_score (report.cpp:7-14)."""
    s = ctypes.c_double(0.0)
    st = lib().fsil_assemble_score(a, b, ctypes.byref(s))
    if st != OK:
        raise ValueError(f"assemble_score: negative mean distance (a={a}, b={b})")
    return s.value


def compare(X, labels, metric="sqeuclid", rtol=1e-9, atol=1e-12, inject_fault=0.0, device: int = 0) -> dict:
    """The reference's `compare` (tools/main.cpp:62-108) on the GPU: the fast engine against
    the naive Theta(N^2 D) engine; every a_i, b_i, s_i must satisfy |fast - naive| <= atol +
    rtol |naive|.  `inject_fault` perturbs the fast s_i (the reference's test hook).  The
    reference's defaults (1e-9, 1e-12) are fp64-vs-fp64; this fast engine certifies
    |ds_i| <= 1e-5 absolute, so GPU compares use atol = 1e-5 and
    rtol ~ 1e-4 (a_i, b_i are certified to ~1e-5 relative)."""
    ctx = default_context(device)
    fast = ctx.silhouette(X, labels, metric)
    naive = ctx.silhouette_naive(X, labels, metric)
    fs = fast.s + inject_fault
    max_abs, max_rel, within = 0.0, 0.0, True
    for got, ref in ((fast.a, naive.a), (fast.b, naive.b), (fs, naive.s)):
        dev = np.abs(got - ref)
        max_abs = max(max_abs, float(dev.max(initial=0.0)))
        nz = ref != 0
        if nz.any():
            max_rel = max(max_rel, float((dev[nz] / np.abs(ref[nz])).max()))
        within = within and bool(np.all(dev <= atol + rtol * np.abs(ref)))
    return {"fast_mean": fast.mean, "naive_mean": naive.mean, "max_abs_deviation": max_abs,
            "max_rel_deviation": max_rel, "within": within, "rtol": rtol, "atol": atol,
            "fast_wall_ms": fast.wall_time_ms, "naive_wall_ms": naive.wall_time_ms}
