#!/usr/bin/env python
"""Benchmark of the B200 linear-time Silhouette hot path (BASELINE.json metric:
Silhouette points/sec at 1/2/4/8 B200, % of roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one whole Silhouette of the workload: densify + cluster aggregation +
scoring + fp64 refinement + deterministic mean (fsil_silhouette_device, inputs
resident in HBM).  Default workload: BASELINE.json configs[1] (C2: cosine,
N=1,000,000, D=64, K=20, fp32).  Multi-GPU (torchrun): each rank holds a
config-sized shard (weak scaling; global N = N_config x world) and the ranks
exchange the dictionary, the K x (D+1) statistics and the scalar sum over NCCL.

Prints ONE JSON line on rank 0.  The `--impl reference` arm times the CPU
restatement of the reference path (oracle/, the reference itself cannot be
compiled here: SURVEY.md 8c) on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_ORDER = ["C1", "C2", "C3", "C4", "C5"]
METRIC = "Silhouette points/sec (N·K dist-evals/s) at 1/2/4/8 B200; % of roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=CONFIG_ORDER)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="auto", choices=["auto", "ffma", "tcgen05", "fp64"])
    ap.add_argument("--n", type=int, default=None, help="override N (parity/debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU protocol (NCCL exchanges) even on one rank (path check)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def bytes_per_point(d):
    # read x (4D) + label (4); write s (8) + neighbour (4)
    return 4 * d + 16


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_baseline(X, L, metric, max_rows, trials=3):
    """CPU restatement of the reference (oracle/, TEST INFRASTRUCTURE) on this host's
    cores: the reference's own run_two_phase window, best of 3 (bench.cpp:72-79)."""
    import oracle

    n = min(X.shape[0], max_rows)
    Xs, Ls = np.ascontiguousarray(X[:n]), np.ascontiguousarray(L[:n])
    cores = os.cpu_count() or 1
    best = None
    for _ in range(trials):
        r = oracle.silhouette(Xs, Ls, metric, "fast", shards=cores)
        best = r.wall_ms if best is None else min(best, r.wall_ms)
    return {"value": n / (best / 1e3), "unit": "points/s", "cores": cores, "kind": "port",
            "sample": f"rows [0,{n}) of the workload, full aggregation+scoring+mean window "
                      f"(engine.hpp:107-113), best of {trials}", "ms": best}


def sample_rows(cfg, d, k):
    # bound the CPU sample to ~10-30 s of fp64 work at ~1 GFLOP/s/core x cores
    cores = os.cpu_count() or 1
    budget_flops = 15e9 * cores
    per_row = 2.0 * k * d + 6 * d
    return int(max(2000, min(budget_flops / per_row, 5_000_000)))


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2303_14102_b200.datagen import CONFIGS

    cid, metric, N, D, K, seed = CONFIGS[a.config]
    N = a.n or N

    if a.impl == "reference":
        if rank != 0:
            return 0
        from paper_2303_14102_b200 import datagen
        import torch
        rows = min(N, sample_rows(a.config, D, K))
        X, L, _ = datagen.generate_host(a.config, n=N if N <= 5_000_000 else rows)
        X, L = X[:rows], L[:rows]
        import oracle
        cores = os.cpu_count() or 1
        for _ in range(max(a.warmup, 0)):
            oracle.silhouette(X, L, metric, "fast", shards=cores)
        times = []
        for _ in range(a.steps):
            times.append(oracle.silhouette(X, L, metric, "fast", shards=cores).wall_ms)
        ms = float(np.mean(times))
        val = rows / (ms / 1e3)
        out = {"metric": METRIC, "value": val, "unit": "points/s", "n_gpus": world,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "impl": "reference",
               "config": {"workload": f"{a.config} ({metric}, N={N}, D={D}, K={K}); CPU step = "
                                      f"rows [0,{rows})", "global_batch": rows, "seq_len": D,
                          "parallelism": f"{cores} host threads (std::thread, engine.cpp:34-55)"},
               "cpu_baseline": {"value": val, "unit": "points/s", "cores": cores, "kind": "port",
                                "sample": f"rows [0,{rows}) of {a.config}, run_two_phase window"},
               "e2e": {"value": val, "unit": "points/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0},
               "gpu_launches": 0}
        print(json.dumps(out))
        return 0

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or a.sharded
    if sharded:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2303_14102_b200 import Context, PATH_AUTO, PATH_FFMA, PATH_TCGEN05
    from paper_2303_14102_b200.api import PATH_FP64
    from paper_2303_14102_b200 import datagen
    from paper_2303_14102_b200.distributed import compute_silhouette_sharded

    X, L, _ = datagen.generate_device(a.config, n=N, seed=seed + 7919 * rank)
    torch.cuda.synchronize()
    ctx = Context(local)
    ctx.set_path({"auto": PATH_AUTO, "ffma": PATH_FFMA, "tcgen05": PATH_TCGEN05,
                  "fp64": PATH_FP64}[a.path])
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    s = torch.empty(N, dtype=torch.float64, device=dev)
    nb = torch.empty(N, dtype=torch.int32, device=dev)
    n_global = N * world

    def step():
        if not sharded:
            return ctx.silhouette_device(X, L, metric, s=s, neighbour=nb)[0]
        return compute_silhouette_sharded(ctx, metric, X, L, rank * N, n_global, s=s, neighbour=nb)

    for _ in range(max(a.warmup, 3)):
        mean = step()
    torch.cuda.synchronize()

    # per-kernel timing pass (CUDA events inside libfsil on the same stream) for the roofline
    ctx.set_timing(True)
    phase = {"densify": [], "aggregate": [], "score": [], "score_kernel": [], "refine": [], "finalize": []}
    for _ in range(3):
        step()
        st = ctx.stats()
        for k_ in phase:
            phase[k_].append(st["ms_" + k_])
    ctx.set_timing(False)
    launches_per_step = ctx.stats()["kernel_launches"]

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(a.steps):
        mean = step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / a.steps
    if sharded:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n_global / (ms / 1e3)
    st = ctx.stats()

    # roofline of the dominant kernel (the scoring pass)
    hbm, tflops, peak_kind = measured_peaks()
    score_ms = float(np.median(phase["score_kernel"]))  # the scoring kernel alone (ev on its stream)
    bpp = bytes_per_point(D)
    achieved = (N * bpp) / (score_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_{a.config}_score_summary.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic,
                "kernel": "scoring kernel alone (score_tc / score_ffma; operand prep excluded)", "peak_source": peak_kind,
                "algorithmic_bytes_per_point": bpp, "points_per_launch": N,
                "launch_ms": score_ms}

    # end-to-end through the public host entry (pinned host buffers, H2D + D2H in the window)
    e2e = None
    if world == 1 and not a.no_e2e:
        hX = torch.empty((N, D), dtype=torch.float32, pin_memory=True)
        hL = torch.empty(N, dtype=torch.int32, pin_memory=True)
        hX.copy_(X)
        hL.copy_(L)
        hs = torch.empty(N, dtype=torch.float64, pin_memory=True)
        hnb = torch.empty(N, dtype=torch.int32, pin_memory=True)
        import ctypes
        from paper_2303_14102_b200.api import lib, metric_code
        mean_c, k_c = ctypes.c_double(), ctypes.c_int32()

        def host_step():
            rc = lib().fsil_silhouette(ctx._h, metric_code(metric), hX.data_ptr(), hL.data_ptr(), N, D,
                                       hs.data_ptr(), hnb.data_ptr(), None, None, None,
                                       ctypes.byref(mean_c), ctypes.byref(k_c), None)
            if rc != 0:
                raise RuntimeError(lib().fsil_last_error(ctx._h).decode())

        for _ in range(3):
            host_step()
        e_steps = max(3, min(a.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(e_steps):
            host_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / e_steps
        e2e = {"value": N / (e_ms / 1e3), "unit": "points/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": N * D * 4 + N * 4, "d2h_bytes_per_step": N * 12 + 8,
               "api": "fsil_silhouette (C ABI, host buffers)", "mean": mean_c.value}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        rows = min(N, sample_rows(a.config, D, K))
        cpu = cpu_baseline(X[:rows].cpu().numpy(), L[:rows].cpu().numpy(), metric, rows)

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
               "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": ms,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic",
               "config": {"workload": f"{a.config}: {metric}, N={N} per GPU, D={D}, K={K}, fp32 "
                                      f"features, int32 labels (BASELINE.json configs[{cid - 1}])",
                          "global_batch": n_global, "seq_len": D, "parallelism": f"dp{world}",
                          "l2": f"inputs larger than L2 ({N * D * 4 / 1e6:.0f} MB X per GPU)",
                          "path": ["", "ffma", "tcgen05", "fp64"][st["path"]],
                          "agg_path": ["", "warp-private smem", "label-sorted", "two-phase batches (warp-private smem)"][st["agg_path"]]},
               "dist_evals_per_s": value * K, "mean_silhouette": mean,
               "refined_rows": st["flagged_rows"],
               "phases_ms": {k_: float(np.median(v)) for k_, v in phase.items()},
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(launches_per_step) * a.steps, "clocks": clk}
        print(json.dumps(out))
    if sharded:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
