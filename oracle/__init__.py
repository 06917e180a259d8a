"""TEST INFRASTRUCTURE ONLY: ctypes binding of the CPU restatement of the
reference fastsil hot path (oracle/fsil_oracle.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this package.  It is the parity checker
and the CPU baseline, never the thing measured or shipped.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfsil_oracle.so")
_REF_PATH = os.path.join(_HERE, "_ref", "libfsil_ref.so")
_REF_SRC = "/root/reference/proj"
_lib = None
_ref_lib = None

SQEUCLID, COSINE, EUCLID = 0, 1, 2
FAST, NAIVE = 0, 1
METRICS = {"sqeuclid": SQEUCLID, "squared_euclidean": SQEUCLID, "cosine": COSINE,
           "euclid": EUCLID, "euclidean": EUCLID}


class OracleValidationError(ValueError):
    """fastsil::ValidationError (types.hpp:41-44)."""


class OracleInvalidArgument(ValueError):
    """std::invalid_argument raised by the reference."""


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _LIB_PATH


def build_ref(force: bool = False):
    """oracle/_ref/libfsil_ref.so: the reference's own sources compiled against the Eigen
    shim (oracle/Makefile `ref`).  Built only where /root/reference exists (this
    container); elsewhere the prebuilt library that travelled with the snapshot is used.
    Returns the path, or None when neither is available."""
    if os.path.isdir(_REF_SRC) and (force or not os.path.exists(_REF_PATH)):
        subprocess.run(["make", "-C", _HERE, "-s", "ref"], check=True)
    return _REF_PATH if os.path.exists(_REF_PATH) else None


def _bind_common(L, prefix):
    P = ctypes.c_void_p
    i64, i32, sz, cp = ctypes.c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.c_char_p
    for name in ("silhouette_f32", "silhouette"):
        getattr(L, f"{prefix}_{name}").argtypes = [i32, i32, P, P, i64, i64, i32, P, P, P, P, P, P, P,
                                                   P, P, cp, sz]
    getattr(L, f"{prefix}_plan_shards").argtypes = [i64, i32, P, P, cp, sz]
    getattr(L, f"{prefix}_assemble_score").argtypes = [ctypes.c_double, ctypes.c_double, P, cp, sz]
    getattr(L, f"{prefix}_default_shards").restype = i32


def ref_lib():
    """The reference library (oracle/_ref), or None if it is not built."""
    global _ref_lib
    if _ref_lib is None:
        path = build_ref()
        if path is None:
            return None
        L = ctypes.CDLL(path)
        _bind_common(L, "ref")
        P = ctypes.c_void_p
        i64, sz, cp = ctypes.c_int64, ctypes.c_size_t, ctypes.c_char_p
        L.ref_generate_blobs.argtypes = [i64, i64, i64, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                         P, P, cp, sz]
        L.ref_read_csv_text.argtypes = [cp, ctypes.c_char, ctypes.c_int, cp, ctypes.c_int, P, P, P, P, cp, sz,
                                        cp, sz]
        L.ref_score_report.argtypes = [ctypes.c_int, P, P, i64, i64, ctypes.c_int, cp, sz, P, cp, sz]
        _ref_lib = L
    return _ref_lib


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, dbl, sz, cp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t, ctypes.c_char_p
        L.orc_silhouette_f32.argtypes = [i32, i32, P, P, i64, i64, i32, P, P, P, P, P, P, P, P, P, cp, sz]
        L.orc_silhouette.argtypes = [i32, i32, P, P, i64, i64, i32, P, P, P, P, P, P, P, P, P, cp, sz]
        L.orc_aggregate_f32.argtypes = [i32, P, P, i64, i64, i32, P, P, P, P, cp, sz]
        L.orc_aggregate_dense_f32.argtypes = [i32, P, P, i64, i64, i32, i32, P, P, P, cp, sz]
        L.orc_score_rows_f32.argtypes = [i32, P, P, i64, i64, i32, P, P, P, P, i64, P, P, P, P, cp, sz]
        L.orc_score_rows_mt_f32.argtypes = [i32, P, P, i64, i64, i32, P, P, P, P, i64, i32, P, P, P, P, cp, sz]
        L.orc_plan_shards.argtypes = [i64, i32, P, P, cp, sz]
        L.orc_assemble_score.argtypes = [dbl, dbl, P, cp, sz]
        L.orc_default_shards.restype = i32
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, err):
    if rc == 0:
        return
    msg = err.value.decode()
    if rc == 2:
        raise OracleValidationError(msg)
    if rc == 3:
        raise OracleInvalidArgument(msg)
    raise RuntimeError(f"oracle error {rc}: {msg}")


@dataclass
class OracleReport:
    a: np.ndarray
    b: np.ndarray
    s: np.ndarray
    own: np.ndarray
    neighbour: np.ndarray
    mean: float
    k: int
    dense_to_raw: np.ndarray
    wall_ms: float


def silhouette(X, labels, metric="sqeuclid", engine="fast", shards=0, reference=False) -> OracleReport:
    """compute_silhouette(validate_and_densify(X, labels), ...) (engine.cpp:76-92).
    reference=True runs the reference's own compiled code (oracle/_ref) instead of the
    restatement; both share this signature."""
    m = METRICS[metric] if isinstance(metric, str) else int(metric)
    e = NAIVE if engine == "naive" else FAST
    X = np.ascontiguousarray(X)
    n = X.shape[0]
    d = X.shape[1] if X.ndim == 2 else 0
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    out = [np.zeros(n) for _ in range(3)] + [np.zeros(n, np.int32) for _ in range(2)]
    mean, wall = ctypes.c_double(0), ctypes.c_double(0)
    k = ctypes.c_int32(0)
    d2r = np.zeros(max(n, 1), np.int32)
    err = ctypes.create_string_buffer(512)
    L, pre = (ref_lib(), "ref") if reference else (lib(), "orc")
    if L is None:
        raise RuntimeError("oracle/_ref/libfsil_ref.so is not built (needs /root/reference)")
    if X.dtype not in (np.float32, np.float64):
        X = X.astype(np.float64)
    fn = getattr(L, f"{pre}_silhouette_f32" if X.dtype == np.float32 else f"{pre}_silhouette")
    rc = fn(m, e, _ptr(X), _ptr(labels), n if labels.shape[0] == n else labels.shape[0], d, shards,
            *[_ptr(o) for o in out], ctypes.byref(mean), ctypes.byref(k), _ptr(d2r),
            ctypes.byref(wall), err, 512)
    _check(rc, err)
    return OracleReport(out[0], out[1], out[2], out[3], out[4], mean.value, k.value,
                        d2r[: k.value].copy(), wall.value)


def aggregate(X, labels, metric="sqeuclid", shards=0):
    """Merged phase-1 statistics (engine.hpp:50-80): (counts, sums[K,D], psi|None)."""
    m = METRICS[metric] if isinstance(metric, str) else int(metric)
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, d = X.shape
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    kmax = len(np.unique(labels))
    counts = np.zeros(kmax, np.int64)
    sums = np.zeros((kmax, d))
    psi = np.zeros(kmax)
    k = ctypes.c_int32(0)
    err = ctypes.create_string_buffer(512)
    rc = lib().orc_aggregate_f32(m, _ptr(X), _ptr(labels), n, d, shards, _ptr(counts), _ptr(sums),
                                 _ptr(psi), ctypes.byref(k), err, 512)
    _check(rc, err)
    return counts, sums, (psi if m == SQEUCLID else None)


def first_appearance(labels):
    """Dense ids by first appearance (dataset.cpp:41-51) without strings: (dense, raw_in_order)."""
    labels = np.asarray(labels)
    uniq, first, inv = np.unique(labels, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.shape[0])
    return rank[inv].astype(np.int32), uniq[order]


def aggregate_dense(X, dense, k, metric="sqeuclid", shards=0):
    """Merged phase-1 statistics over already-dense labels -> (counts, sums[K,D], psi|None)."""
    m = METRICS[metric] if isinstance(metric, str) else int(metric)
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, d = X.shape
    dense = np.ascontiguousarray(dense, dtype=np.int32)
    counts = np.zeros(k, np.int64)
    sums = np.zeros((k, d))
    psi = np.zeros(k)
    err = ctypes.create_string_buffer(512)
    rc = lib().orc_aggregate_dense_f32(m, _ptr(X), _ptr(dense), n, d, k, shards, _ptr(counts),
                                       _ptr(sums), _ptr(psi), err, 512)
    _check(rc, err)
    return counts, sums, (psi if m == SQEUCLID else None)


def score_rows(X, dense, counts, sums, psi, rows, metric="sqeuclid", threads=1, want_ab=True):
    """score_range on rows (None = all) against global stats -> (a, b, s, neighbour);
    threads=0 uses every host core.  want_ab=False returns a, b as None (saves 16 B/row)."""
    m = METRICS[metric] if isinstance(metric, str) else int(metric)
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, d = X.shape
    dense = np.ascontiguousarray(dense, dtype=np.int32)
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    sums = np.ascontiguousarray(sums, dtype=np.float64)
    psi_a = None if psi is None else np.ascontiguousarray(psi, dtype=np.float64)
    rows = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    mm = n if rows is None else rows.shape[0]
    a, b = (np.zeros(mm), np.zeros(mm)) if want_ab else (None, None)
    s = np.zeros(mm)
    nb = np.zeros(mm, np.int32)
    err = ctypes.create_string_buffer(512)
    rc = lib().orc_score_rows_mt_f32(m, _ptr(X), _ptr(dense), n, d, counts.shape[0], _ptr(counts),
                                     _ptr(sums), _ptr(psi_a), _ptr(rows), mm, threads, _ptr(a), _ptr(b),
                                     _ptr(s), _ptr(nb), err, 512)
    _check(rc, err)
    return a, b, s, nb


def plan_shards(n, w, reference=False):
    """plan_shards (engine.cpp:8-25) -> list of (begin, end)."""
    ranges = np.zeros(2 * max(1, min(max(w, 1), max(n, 1))), np.int64)
    ns = ctypes.c_int(0)
    err = ctypes.create_string_buffer(512)
    fn = ref_lib().ref_plan_shards if reference else lib().orc_plan_shards
    rc = fn(n, w, _ptr(ranges), ctypes.byref(ns), err, 512)
    _check(rc, err)
    return [(int(ranges[2 * i]), int(ranges[2 * i + 1])) for i in range(ns.value)]


def assemble_score(a, b, reference=False):
    s = ctypes.c_double(0)
    err = ctypes.create_string_buffer(512)
    fn = ref_lib().ref_assemble_score if reference else lib().orc_assemble_score
    rc = fn(a, b, ctypes.byref(s), err, 512)
    _check(rc, err)
    return s.value


def default_shards():
    return lib().orc_default_shards()


def ref_generate_blobs(n, d, k, seed, spread=1.0, separation=8.0):
    """The reference's generate_blobs (blobs.cpp:25-54) -> (X fp64 [n,d], dense labels)."""
    X = np.zeros((n, d))
    L = np.zeros(n, np.int32)
    err = ctypes.create_string_buffer(512)
    _check(ref_lib().ref_generate_blobs(n, d, k, spread, separation, seed, _ptr(X), _ptr(L), err, 512), err)
    return X, L


def ref_read_csv_text(text, delimiter=",", label_index=-1, label_name="", has_header=None):
    """The reference's read_csv_text (csv.cpp:54-159) -> (X fp64, dense labels, names)."""
    L = ref_lib()
    t = text.encode()
    n, d = ctypes.c_int64(0), ctypes.c_int64(0)
    err = ctypes.create_string_buffer(1024)
    hh = -1 if has_header is None else int(bool(has_header))
    args = (t, delimiter.encode(), label_index, label_name.encode(), hh)
    _check(L.ref_read_csv_text(*args, ctypes.byref(n), ctypes.byref(d), None, None, None, 0, err, 1024), err)
    X = np.zeros((n.value, d.value))
    lab = np.zeros(n.value, np.int32)
    names = ctypes.create_string_buffer(1 << 20)
    _check(L.ref_read_csv_text(*args, ctypes.byref(n), ctypes.byref(d), _ptr(X), _ptr(lab), names, 1 << 20,
                               err, 1024), err)
    return X, lab, names.value.decode().split("\n")[:-1]


def ref_score_report(X, labels, metric="sqeuclid", fmt="csv"):
    """compute_silhouette(..., shards=1) then write_report (report_io.cpp:53-68) -> text."""
    m = METRICS[metric] if isinstance(metric, str) else int(metric)
    X = np.ascontiguousarray(X, dtype=np.float64)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    n, d = X.shape
    L = ref_lib()
    ln = ctypes.c_size_t(0)
    err = ctypes.create_string_buffer(1024)
    f = 1 if fmt == "jsonl" else 0
    _check(L.ref_score_report(m, _ptr(X), _ptr(labels), n, d, f, None, 0, ctypes.byref(ln), err, 1024), err)
    buf = ctypes.create_string_buffer(ln.value + 1)
    _check(L.ref_score_report(m, _ptr(X), _ptr(labels), n, d, f, buf, ln.value + 1, ctypes.byref(ln), err, 1024),
           err)
    return buf.value.decode()
