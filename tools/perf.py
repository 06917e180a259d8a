"""Per-config timing of the libfsil pipeline on one GPU (builder tool; not a bench line).

    python tools/perf.py C2 C3:400000 C5 [--path 2] [--reps 5] [--out gpurun_out/perf.json]

For each config: device-resident inputs from the seeded generators, warm-up, CUDA-event
time per call, then one timed call with libfsil's per-phase events (fsil_stats)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_14102_b200 import Context, datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default="gpurun_out/perf.json")
a = ap.parse_args()
res = {}
for cfg in a.configs:
    name, n = cfg.split(":") if ":" in cfg else (cfg, None)
    ctx = Context(0)
    ctx.set_path(a.path)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    X, L, metric = datagen.generate_device(name, n=int(n) if n else None)
    N = X.shape[0]
    s = torch.empty(N, dtype=torch.float64, device="cuda")
    nb = torch.empty(N, dtype=torch.int32, device="cuda")
    for _ in range(2):
        ctx.silhouette_device(X, L, metric, s=s, neighbour=nb)
    reps = 2 if name == "C5" and n is None else a.reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        mean, k = ctx.silhouette_device(X, L, metric, s=s, neighbour=nb)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ctx.set_timing(True)
    ctx.silhouette_device(X, L, metric, s=s, neighbour=nb)
    st = ctx.stats()
    ctx.set_timing(False)
    r = dict(ms=ms, pts_per_s=N / ms * 1e3, mean=mean, **st)
    res[cfg] = r
    print(cfg, json.dumps({k_: (round(v, 4) if isinstance(v, float) else v) for k_, v in r.items()}), flush=True)
    del X, L, s, nb
    ctx.close()
    torch.cuda.empty_cache()
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump(res, open(a.out, "w"), indent=1)
