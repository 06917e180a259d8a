"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: BASELINE.json names none, and the paper's
129-feature set is proprietary.  Each config is a fully specified seeded
distribution; the same bytes are fed to libfsil and to the CPU oracle.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .api import DATAGEN_PATH, FsilError, ERR_INTERNAL

# name -> (generator config id, metric, N, D, K, seed)
CONFIGS = {
    "C1": (1, "sqeuclid", 100_000, 16, 8, 2303141021),
    "C2": (2, "cosine", 1_000_000, 64, 20, 2303141022),
    "C3": (3, "sqeuclid", 10_000_000, 128, 100, 2303141023),
    "C4": (4, "sqeuclid", 100_000_000, 32, 1000, 2303141024),
    "C5": (5, "cosine", 40_000_000, 768, 4096, 2303141025),
}

_lib = None


def _dl():
    global _lib
    if _lib is None:
        if not os.path.exists(DATAGEN_PATH):
            raise FsilError(ERR_INTERNAL, f"{DATAGEN_PATH} is not built")
        L = ctypes.CDLL(DATAGEN_PATH)
        P = ctypes.c_void_p
        L.fsilgen_blobs_host.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_uint64, P, P]
        L.fsilgen_device.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_uint64, P, P, P, ctypes.c_char_p, ctypes.c_size_t]
        L.fsilgen_device_rows.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, P, P, P,
                                          ctypes.c_char_p, ctypes.c_size_t]
        _lib = L
    return _lib


def blobs(n, d, k, seed, spread=1.0, separation=10.0):
    """The reference's generate_blobs recipe (blobs.cpp:25-54), fp64 rounded to fp32."""
    X = np.empty((n, d), np.float32)
    L = np.empty(n, np.int32)
    rc = _dl().fsilgen_blobs_host(n, d, k, spread, separation, seed, X.ctypes.data, L.ctypes.data)
    if rc != 0:
        raise ValueError("blob spec invalid")
    return X, L


def generate_device(config: str, n=None, d=None, k=None, seed=None, device=0, rows=None):
    """Generate a config on the GPU -> (X [n,d] float32 cuda tensor, labels [n] int32).
    rows=(begin, end): only those rows of the n-row dataset (one rank's shard of a global
    dataset, byte-identical to the same rows of the whole)."""
    import torch

    cid, metric, N, D, K, S = CONFIGS[config]
    n, d, k, seed = n or N, d or D, k or K, S if seed is None else seed
    dev = torch.device("cuda", device)
    b, e = rows if rows is not None else (0, n)
    if cid == 1:
        X, L = blobs(n, d, k, seed)
        return torch.from_numpy(X[b:e]).to(dev), torch.from_numpy(L[b:e]).to(dev), metric
    X = torch.empty((e - b, d), dtype=torch.float32, device=dev)
    L = torch.empty(e - b, dtype=torch.int32, device=dev)
    err = ctypes.create_string_buffer(256)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = _dl().fsilgen_device_rows(cid, n, b, e - b, d, k, seed, X.data_ptr(), L.data_ptr(), stream, err, 256)
    if rc != 0:
        raise FsilError(ERR_INTERNAL, err.value.decode())
    return X, L, metric


def generate_host(config: str, n=None, d=None, k=None, seed=None, device=0):
    """Same bytes as generate_device, copied to host numpy arrays."""
    X, L, metric = generate_device(config, n, d, k, seed, device)
    return X.cpu().numpy(), L.cpu().numpy(), metric
