#!/usr/bin/env python
"""Benchmark of the B200 linear-time Silhouette hot path (BASELINE.json metric:
Silhouette points/sec at 1/2/4/8 B200, % of roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--also C4]
                    [--impl ours|reference]

A step is one whole Silhouette of the workload: densify + cluster aggregation +
tensor-core neighbour nomination + fp64 refinement/exact pass + deterministic
mean, on HBM-resident inputs.  Default workload: BASELINE.json configs[4] (C5:
cosine, N=40,000,000, D=768, K=4,096, fp32, 123 GB) -- the largest configuration
one B200 holds; C4 (the 100M-point config of the scaling target) is measured in
the same run and reported under "also".

Scaling is STRONG: the global dataset is fixed; with N GPUs each rank generates its
plan_shards (engine.cpp:8-25) rows of the one global dataset (byte-identical to those
rows of the whole) and the ranks run the sharded protocol (dictionary all-gather,
K x (D+2) fp64 all-reduce, scalar all-reduce over NCCL).  `--gpus N` without
WORLD_SIZE in the environment re-launches itself under torch.distributed.run.

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's own CPU
code for the path -- its .cpp files compiled unmodified against the Eigen shim
(oracle/_ref, built by oracle/Makefile `ref`; kind "reference") -- on this host's cores;
where that library is absent it falls back to the bit-identical restatement (oracle/,
kind "port").  Both are test infrastructure, never the measured product.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
TENSOR_CONFIGS = {"C4", "C5"}  # FLOP-bound at P_tc; C1-C3 HBM-bound


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", choices=CONFIG_ORDER)
    ap.add_argument("--also", default=None, help="comma-separated secondary configs (default: C4 with C5)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="auto", choices=["auto", "ffma", "tcgen05", "fp64"])
    ap.add_argument("--n", type=int, default=None, help="override N (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU protocol (NCCL exchanges) even on one rank (path check)")
    a = ap.parse_args()
    if a.also is None:
        a.also = "C4" if a.config == "C5" else ""
    a.also = [c for c in a.also.split(",") if c and c != a.config]
    return a


def maybe_relaunch(a) -> int | None:
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) with this same command."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return {"hbm": float(j["hbm_gbs"]), "tc_burst": float(j["bf16_tflops"]),
                "tc_sustained": float(j.get("bf16_tflops_sustained", j["bf16_tflops"])), "src": "measured"}
    # B200_PROFILING.md fallback
    return {"hbm": 6650.0, "tc_burst": 1590.0, "tc_sustained": 1590.0, "src": "fallback"}


def bytes_per_point(d):
    # read x (4D) + label (4); write s (8) + neighbour (4)
    return 4 * d + 16


def plan_shards(n, w):
    """plan_shards (engine.cpp:8-25): w' = min(w, n) contiguous ranges, the first n mod w'
    one row longer."""
    w = max(1, min(w, n))
    base, extra = divmod(n, w)
    out, b = [], 0
    for i in range(w):
        e = b + base + (1 if i < extra else 0)
        out.append((b, e))
        b = e
    return out


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
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


def cpu_sample_rows(config, d, k):
    """Rows of the CPU sample: about 3 s of the reference path's fp64 work on this host
    (per-row cost 2KD + O(D), independent of N -- PAPER.md:238-249)."""
    cores = os.cpu_count() or 1
    budget_flops = 3.0e9 * cores  # ~1.3 GFLOP/s/core measured for the scalar port, x ~2.3 s
    per_row = 2.0 * k * d + 6 * d
    rows = int(budget_flops / per_row)
    return int(max(2 * k, min(rows, 5_000_000)))


def cpu_sample(config, n_full):
    """The CPU sample of a workload: the config's own generator at N = M rows (same K, D
    and value distributions; every cluster present for C3-C5's size rules), or the first
    M rows when the config's N is small enough to generate whole."""
    from paper_2303_14102_b200 import datagen
    cid, metric, N, D, K, seed = datagen.CONFIGS[config]
    rows = min(n_full, cpu_sample_rows(config, D, K))
    if n_full <= 5_000_000:
        X, L, _ = datagen.generate_host(config, n=n_full)
        X, L = X[:rows], L[:rows]
        how = f"rows [0,{rows}) of {config}"
    else:
        X, L, _ = datagen.generate_host(config, n=rows)
        how = (f"{config} recipe at N={rows} (D={D}, K={K}); per-row cost 2KD is independent of N, "
               f"so points/s extrapolates to N={n_full}")
    return X, L, metric, rows, how


def cpu_impl():
    """(kind, run) for the CPU arm: the reference's own compiled code (oracle/_ref) when
    present, else the restatement that tests/test_reference_pin.py pins to it bit for bit."""
    import oracle
    ref = oracle.ref_lib() is not None
    kind = "reference" if ref else "port"
    return kind, lambda X, L, metric, cores: oracle.silhouette(X, L, metric, "fast", shards=cores, reference=ref)


def cpu_baseline(config, n_full, trials=3):
    """The reference's CPU path (oracle/_ref, or the restatement; TEST INFRASTRUCTURE) on
    this host's cores: the reference's own run_two_phase window (engine.hpp:107-113),
    best of 3 (bench.cpp:72-79)."""
    kind, run = cpu_impl()
    X, L, metric, rows, how = cpu_sample(config, n_full)
    cores = os.cpu_count() or 1
    best = None
    for _ in range(trials):
        r = run(X, L, metric, cores)
        best = r.wall_ms if best is None else min(best, r.wall_ms)
    return {"value": rows / (best / 1e3), "unit": "points/s", "cores": cores, "kind": kind,
            "sample": how + f"; full aggregation+scoring+mean window, best of {trials}", "ms": best}


def reference_arm(a, rank, world):
    """--impl reference: the reference's CPU path (oracle/_ref; else the restatement) on
    this host's cores, rank 0 only, each step a bounded sample of the workload."""
    if rank != 0:
        return 0
    from paper_2303_14102_b200 import datagen
    kind, run = cpu_impl()
    cid, metric, N, D, K, seed = datagen.CONFIGS[a.config]
    N = a.n or N
    X, L, metric, rows, how = cpu_sample(a.config, N)
    cores = os.cpu_count() or 1
    for _ in range(max(a.warmup, 0)):
        run(X, L, metric, cores)
    times = [run(X, L, metric, cores).wall_ms for _ in range(a.steps)]
    ms = float(np.mean(times))
    val = rows / (ms / 1e3)
    out = {"metric": METRIC, "value": val, "unit": "points/s", "n_gpus": world,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": f"{a.config} ({metric}, N={N}, D={D}, K={K}); CPU step = {how}",
                      "global_batch": rows, "seq_len": D,
                      "parallelism": f"{cores} host threads (std::thread, engine.cpp:34-55)"},
           "cpu_baseline": {"value": val, "unit": "points/s", "cores": cores, "kind": kind, "sample": how},
           "e2e": {"value": val, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out))
    return 0


class Runner:
    """One config on this rank: resident shard, timed steps, phase timing, e2e."""

    def __init__(self, a, config, rank, world, local, dev):
        import torch
        from paper_2303_14102_b200 import Context, PATH_AUTO, PATH_FFMA, PATH_TCGEN05, datagen
        from paper_2303_14102_b200.api import PATH_FP64
        self.torch = torch
        self.a, self.config, self.rank, self.world, self.dev = a, config, rank, world, dev
        cid, self.metric, N, self.D, self.K, seed = datagen.CONFIGS[config]
        self.cid = cid
        self.N = (a.n or N) if config == a.config else N
        self.b, self.e = plan_shards(self.N, world)[rank] if rank < min(world, self.N) else (self.N, self.N)
        self.n = self.e - self.b
        self.sharded = world > 1 or a.sharded
        self.X, self.L, _ = datagen.generate_device(config, n=self.N, rows=(self.b, self.e), device=local)
        torch.cuda.synchronize()
        self.ctx = Context(local)
        self.ctx.set_path({"auto": PATH_AUTO, "ffma": PATH_FFMA, "tcgen05": PATH_TCGEN05, "fp64": PATH_FP64}[a.path])
        self.stream = torch.cuda.current_stream(dev)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.s = torch.empty(self.n, dtype=torch.float64, device=dev)
        self.nb = torch.empty(self.n, dtype=torch.int32, device=dev)

    def step(self, X=None, L=None):
        from paper_2303_14102_b200.distributed import compute_silhouette_sharded
        X = self.X if X is None else X
        L = self.L if L is None else L
        if not self.sharded:
            return self.ctx.silhouette_device(X, L, self.metric, s=self.s, neighbour=self.nb)[0]
        return compute_silhouette_sharded(self.ctx, self.metric, X, L, self.b, self.N, s=self.s, neighbour=self.nb)

    def timed(self, steps, fn):
        """max over ranks of the device time of `steps` calls (CUDA events on the stream)."""
        import torch.distributed as dist
        torch = self.torch
        if self.sharded:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(self.stream)
        out = None
        for _ in range(steps):
            out = fn()
        ev1.record(self.stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / steps
        if self.sharded:
            dist.barrier()
            t = torch.tensor([ms], dtype=torch.float64, device=self.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, out

    def run(self, steps, warmup, clocks=None):
        a = self.a
        for _ in range(max(warmup, 3)):
            self.step()
        self.torch.cuda.synchronize()
        # per-kernel timing pass (libfsil's CUDA events on its stream) for the roofline
        self.ctx.set_timing(True)
        phase = {k: [] for k in ("densify", "aggregate", "score", "score_kernel", "refine", "finalize")}
        for _ in range(2):
            self.step()
            st = self.ctx.stats()
            for k_ in phase:
                phase[k_].append(st["ms_" + k_])
        self.ctx.set_timing(False)
        self.st = self.ctx.stats()
        if clocks:
            clocks.start()
            time.sleep(0.3)
        self.ms, self.mean = self.timed(steps, self.step)
        self.clk = clocks.stop() if clocks else None
        self.phases = {k_: float(np.median(v)) for k_, v in phase.items()}
        self.value = self.N / (self.ms / 1e3)
        return self

    def roofline(self):
        pk = measured_peaks()
        score_ms = self.phases["score_kernel"]
        rf = {"kernel": "tensor-core neighbour pass alone (score_tc; operand prep excluded)",
              "peak_source": pk["src"], "points_per_launch": self.n, "launch_ms": score_ms}
        traffic = None
        prof = os.path.join(ROOT, "profiles", f"ncu_{self.config}_score_summary.json")
        if os.path.exists(prof):
            with open(prof) as f:
                j = json.load(f)
            if "dram_bytes_per_point" in j:
                traffic = j["dram_bytes_per_point"] * self.n
                rf["traffic_source"] = f"{os.path.relpath(prof, ROOT)} (ncu --set full, per point x points)"
            else:
                traffic = j.get("dram_bytes_per_launch")
        if self.config in TENSOR_CONFIGS:
            # split-precision rate: m fp16 MMAs per product, the sustained bf16 figure for a
            # kernel inside a long step.  m = 3 (fp16x3) or 2 (the two-level
            # certificate's first level, which scores every row; its three-MMA re-score of
            # the uncertain rows is inside the timed kernel window)
            mmas = int(self.st.get("tc_mmas", 0) or 3)
            peak = pk["tc_sustained"] / mmas
            flops = 2.0 * self.K * self.D * self.n
            achieved = flops / (score_ms / 1e3) / 1e12
            rf.update({"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                       "frac": achieved / peak, "traffic": traffic, "algorithmic_flops_per_point": 2 * self.K * self.D,
                       "mmas_per_product": mmas,
                       "rescored_rows": int(self.st.get("rescored_rows", 0)),
                       "peak_note": f"P_tc = bf16_tflops_sustained / {mmas} (split precision, {mmas} fp16 MMAs "
                                    f"per K step of the pass that scores every row)"})
        else:
            bpp = bytes_per_point(self.D)
            achieved = (self.n * bpp) / (score_ms / 1e3) / 1e9
            rf.update({"bound": "hbm", "achieved": achieved, "peak": pk["hbm"], "unit": "GB/s",
                       "frac": achieved / pk["hbm"], "traffic": traffic, "algorithmic_bytes_per_point": bpp})
        return rf

    def e2e(self, steps):
        """The same metric through the host entry (pinned host X and labels copied in, s and
        neighbour copied out, every step).  The resident device copy is released first so
        the largest config's host entry fits (it stages its own device copy)."""
        import ctypes
        torch = self.torch
        n, D = self.n, self.D
        try:
            hX = torch.empty((n, D), dtype=torch.float32, pin_memory=True)
            hL = torch.empty(n, dtype=torch.int32, pin_memory=True)
            mem = "pinned"
        except RuntimeError:
            hX = torch.empty((n, D), dtype=torch.float32)
            hL = torch.empty(n, dtype=torch.int32)
            mem = "pageable"
        hX.copy_(self.X)
        hL.copy_(self.L)
        hs = torch.empty(n, dtype=torch.float64, pin_memory=mem == "pinned")
        hnb = torch.empty(n, dtype=torch.int32, pin_memory=mem == "pinned")
        torch.cuda.synchronize()
        del self.X, self.L
        torch.cuda.empty_cache()
        if not self.sharded:
            from paper_2303_14102_b200.api import lib, metric_code
            mean_c, k_c = ctypes.c_double(), ctypes.c_int32()
            h = self.ctx._h

            def host_step():
                rc = lib().fsil_silhouette(h, metric_code(self.metric), hX.data_ptr(), hL.data_ptr(), n, D,
                                           hs.data_ptr(), hnb.data_ptr(), None, None, None,
                                           ctypes.byref(mean_c), ctypes.byref(k_c), None)
                if rc != 0:
                    raise RuntimeError(lib().fsil_last_error(h).decode())
                return mean_c.value
            api = "fsil_silhouette (C ABI, host buffers)"
        else:
            dX = torch.empty((n, D), dtype=torch.float32, device=self.dev)
            dL = torch.empty(n, dtype=torch.int32, device=self.dev)

            def host_step():
                dX.copy_(hX, non_blocking=True)
                dL.copy_(hL, non_blocking=True)
                m = self.step(dX, dL)
                hs.copy_(self.s, non_blocking=True)
                hnb.copy_(self.nb, non_blocking=True)
                return m
            api = "compute_silhouette_sharded (host shards copied in/out per step)"
        host_step()
        e_ms, mean = self.timed(steps, host_step)
        return {"value": self.N / (e_ms / 1e3), "unit": "points/s", "ms_per_step": e_ms,
                "h2d_bytes_per_step": (n * D * 4 + n * 4) * self.world,
                "d2h_bytes_per_step": (n * 12 + 8) * self.world, "api": api, "host_memory": mem,
                "steps": steps, "mean": mean}

    def close(self):
        for attr in ("X", "L", "s", "nb"):
            if hasattr(self, attr):
                delattr(self, attr)
        self.ctx.close()
        self.torch.cuda.empty_cache()


def main():
    a = parse()
    rc = maybe_relaunch(a)
    if rc is not None:
        return rc
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return reference_arm(a, rank, world)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or a.sharded:
        dist.init_process_group("nccl", device_id=dev)

    main_r = Runner(a, a.config, rank, world, local, dev)
    main_r.run(a.steps, a.warmup, ClockSampler(local))
    roof = main_r.roofline()
    st = main_r.st
    e2e = None if a.no_e2e else main_r.e2e(max(2, min(a.steps, 5)))
    main_r.close()

    also = {}
    for cfg in a.also:
        r = Runner(a, cfg, rank, world, local, dev).run(a.steps, a.warmup)
        also[cfg] = {"value": r.value, "unit": "points/s", "ms_per_step": r.ms, "global_batch": r.N,
                     "seq_len": r.D, "k": r.K, "metric": r.metric, "mean_silhouette": r.mean,
                     "dist_evals_per_s": r.value * r.K, "phases_ms": r.phases, "roofline": r.roofline(),
                     "refined_rows": r.st["flagged_rows"], "pair_rows": r.st["pair_rows"],
                     "e2e": None if a.no_e2e else r.e2e(max(2, min(a.steps, 5)))}
        r.close()

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a.config, main_r.N)

    if rank == 0:
        from paper_2303_14102_b200 import datagen
        cid = datagen.CONFIGS[a.config][0]
        out = {"metric": METRIC, "value": main_r.value, "unit": "points/s", "n_gpus": world,
               "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": main_r.ms,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic",
               "config": {"workload": f"{a.config}: {main_r.metric}, N={main_r.N} (global, plan_shards rows per "
                                      f"rank), D={main_r.D}, K={main_r.K}, fp32 features, int32 labels "
                                      f"(BASELINE.json configs[{cid - 1}])",
                          "global_batch": main_r.N, "seq_len": main_r.D, "parallelism": f"dp{world} (row shards)",
                          "l2": f"inputs larger than L2 ({main_r.n * main_r.D * 4 / 1e9:.1f} GB X per GPU)",
                          "path": ["", "ffma", "tcgen05", "fp64"][st["path"]],
                          "agg_path": ["", "warp-private smem", "label-sorted", "two-phase batches"][st["agg_path"]]},
               "dist_evals_per_s": main_r.value * main_r.K, "mean_silhouette": main_r.mean,
               "refined_rows": st["flagged_rows"], "pair_rows": st["pair_rows"],
               "phases_ms": main_r.phases, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(st["kernel_launches"]) * a.steps, "clocks": main_r.clk, "also": also}
        print(json.dumps(out))
    if world > 1 or a.sharded:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
