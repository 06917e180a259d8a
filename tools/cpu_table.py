"""the reference's own CPU path (oracle/_ref: the reference .cpp files
compiled against the Eigen shim) on this host's cores, per BASELINE config, with the
reference's run_two_phase window (engine.hpp:105-115) and best of 3 (bench.cpp:72-79).
Configs too large for a full CPU run are timed on a seeded sample of the same recipe (the
per-row cost 2KD + O(D) does not depend on N) and labelled as such.

    python tools/cpu_table.py [--out gpurun_out/cpu_table.json]
"""
import argparse
import json
import os
import platform
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the CPU reference arm)
from paper_2303_14102_b200 import datagen  # noqa: E402

SAMPLES = {"C1": None, "C2": None, "C3": 1_000_000, "C4": 500_000, "C5": 8192}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/cpu_table.json")
    a = ap.parse_args()
    ref = oracle.ref_lib() is not None
    cores = os.cpu_count() or 1
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except (OSError, IndexError):
        model = platform.processor()
    mem = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout.split("\n")[1]
    out = {"kind": "reference" if ref else "port", "cores": cores, "cpu": model, "mem": mem, "configs": {}}
    for name, sample in SAMPLES.items():
        cid, metric, N, D, K, seed = datagen.CONFIGS[name]
        n = N if sample is None else sample
        X, L, _ = datagen.generate_host(name, n=n)
        best = None
        for _ in range(3):
            r = oracle.silhouette(X, L, metric, "fast", shards=cores, reference=ref)
            best = r.wall_ms if best is None else min(best, r.wall_ms)
        pts = n / (best / 1e3)
        row = {"n_timed": n, "n_config": N, "ms": best, "points_per_s": pts,
               "full_config_s_extrapolated": N / pts, "mean_silhouette": r.mean,
               "sample": "full config" if sample is None else f"{name} recipe at N={n}, extrapolated to N={N}"}
        out["configs"][name] = row
        print(name, json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
