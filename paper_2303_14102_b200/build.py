"""In-tree build of the sm_100a libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

    python -m paper_2303_14102_b200.build            # incremental
    python -m paper_2303_14102_b200.build --force

Products (git-ignored, not gpurun-ignored):
    paper_2303_14102_b200/libfsil.so         the product: C ABI of include/fsil.h
    paper_2303_14102_b200/libfsil_datagen.so synthetic config generators (bench/test inputs)
    paper_2303_14102_b200/libfsil_probe.so   tcgen05 accumulation probe (tests only)
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-O3",
         f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]

LIBS = {
    "libfsil.so": ["densify.cu", "aggregate.cu", "score_ffma.cu", "score_tc.cu", "score_tc2.cu", "naive.cu", "finalize.cu",
                   "capi.cu"],
    "libfsil_datagen.so": ["datagen.cu"],
    # test infrastructure: the tcgen05 accumulation probe (tests/test_tc_numerics.py)
    "libfsil_probe.so": ["tc_probe.cu"],
}


def _headers():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + [
        os.path.join(ROOT, "include", "fsil.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src, force):
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    if force or _stale(obj, [src] + _headers()):
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> dict:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted({s for v in LIBS.values() for s in v})
    srcs = [os.path.join(CSRC, s) for s in srcs if os.path.exists(os.path.join(CSRC, s))]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = dict(zip(srcs, ex.map(lambda s: _compile(s, force), srcs)))
    out = {}
    for lib, files in LIBS.items():
        lib_objs = [objs[os.path.join(CSRC, f)] for f in files if os.path.join(CSRC, f) in objs]
        if not lib_objs:
            continue
        target = os.path.join(PKG, lib)
        if force or _stale(target, lib_objs):
            cmd = [NVCC, *ARCH, "-shared", "-o", target, *lib_objs, "-Xcompiler", "-fPIC"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"link failed for {lib}:\n{r.stderr}")
        if verbose:
            print(f"built {target}")
        out[lib] = target
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    try:
        build(force=a.force, verbose=True)
    except RuntimeError as e:
        print(e, file=sys.stderr)
        sys.exit(1)
