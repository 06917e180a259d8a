"""CPU tests of the drop-in boundary: libfsil.so builds for sm_100a, loads, exports
every entry point include/fsil.h declares, and its host-only entries agree with
the oracle.  No kernels are launched here (no GPU in the dev container)."""
import ctypes
import json
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from paper_2303_14102_b200 import api, datagen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fsil.h")).read()
    return sorted(set(re.findall(r"\b(fsil_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = api.lib()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), f"libfsil.so does not export {s}"
    assert set(syms) == set(api.EXPORTS), "api.EXPORTS out of sync with include/fsil.h"
    assert L.fsil_abi_version() == 1


def test_library_is_sm100a_native():
    so = api.LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True,
                          text=True).stdout
    assert "FFMA2" in sass, "packed FFMA2 missing from the FFMA scoring kernel"
    for kern in ("score_ffma_kernel", "score_tc_kernel", "agg_stage_kernel", "agg_warp_kernel",
                 "agg_piece_kernel", "densify_collect_kernel", "refine_kernel"):
        assert kern in sass, kern
    # tcgen05 MMA (UTCHMMA), TMA tensor loads (UTMALDG) and bulk copies (UBLKCP)
    for op in ("UTCHMMA", "UTMALDG", "UBLKCP"):
        assert op in sass, op


def test_host_entries_match_oracle():
    for n, w in ((10, 3), (2, 8), (5, 1), (1000, 7), (7, 7)):
        assert api.plan_shards(n, w) == oracle.plan_shards(n, w)
    for a, b in ((1.0, 16.5), (0.0, 0.0), (2.0, 1.0), (3.0, 3.0), (0.0, 5.0)):
        assert api.assemble_score(a, b) == oracle.assemble_score(a, b)
    with pytest.raises(ValueError):
        api.assemble_score(-1.0, 1.0)
    with pytest.raises(ValueError):
        api.plan_shards(0, 1)


def test_no_cpu_fallback_without_device():
    # fsil_create must fail loudly when there is no usable sm_100 device
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("a GPU is present")
    with pytest.raises(api.FsilError) as e:
        api.Context(0)
    assert e.value.status == api.ERR_CUDA


def test_metric_parsing_mirrors_reference():
    # parse_metric (types.cpp:21-28)
    assert api.metric_code("sqeuclid") == api.SQEUCLID == api.metric_code("squared_euclidean")
    assert api.metric_code("cosine") == api.COSINE
    assert api.metric_code("euclid") == api.EUCLID
    with pytest.raises(api.ValidationError):
        api.metric_code("manhattan")


def test_c1_generator_is_the_reference_blob_recipe():
    # blobs.hpp:13-44 / blobs.cpp:11-54, pinned against a pure-Python restatement
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["blobs_n64_d3_k4_seed42"]
    X, L = datagen.blobs(64, 3, 4, 42, spread=1.0, separation=8.0)
    assert L.tolist() == g["labels"]
    assert np.array_equal(X, np.array(g["X"]).astype(np.float32))


def test_configs_match_baseline_json():
    cfg = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert len(cfg) == 5
    for name, (cid, metric, n, d, k, _) in datagen.CONFIGS.items():
        text = cfg[cid - 1].replace(",", "")
        assert f"N={n}" in text and f"D={d}" in text and f"K={k}" in text
        assert ("Cosine" in text) == (metric == "cosine")
