"""Summarise ncu captures into the small JSON / markdown files committed under profiles/.

Run here (no GPU needed) on what a gpurun call brought back:

    python profiles/summarize_ncu.py --round r01 gpurun_out/r01_*.ncu-rep \
        --launches gpurun_out/launches_bench_c2.csv

For each `--set full` report it writes profiles/<round>_<name>.json with the metrics
the roofline discussion in DESIGN.md cites (duration, DRAM bytes, throughputs, tensor
pipe activity, occupancy, L2 hit rate).  The C2 scoring capture also refreshes
profiles/ncu_C2_score_summary.json, whose dram_bytes_per_launch bench.py reports as
roofline.traffic.  The launch list (the `--metrics gpu__time_duration.sum` pass over
bench.py) becomes a per-kernel table with each kernel's share of the step.
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
NCU = "/usr/local/cuda/bin/ncu"

METRICS = {
    "duration": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "tensor_smem_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "inst_executed": "smsp__inst_executed.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "s": 1, "second": 1, "%": 1, "": 1,
         "register/thread": 1, "inst": 1, "block": 1, "thread": 1, "Kbyte/block": 1e3, "byte/block": 1}
# synthetic-data generation (datagen.cu) runs once before the timed steps: not part of a step
SETUP_KERNELS = ("centres_kernel", "uniform_labels_kernel", "points_kernel", "nearest_kernel",
                 "zipf_labels_kernel", "dirichlet_labels_kernel", "shuffle_kernel", "labels_kernel")


def raw(rep, row=0):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2 + row]
    return head, units, vals


def n_kernels(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    return len(list(csv.reader(io.StringIO(out)))) - 2


def summarise(rep, row=0):
    head, units, vals = raw(rep, row)
    col = {h: i for i, h in enumerate(head)}
    res = {"report": os.path.basename(rep), "kernel": vals[col["Kernel Name"]]}
    for key, m in METRICS.items():
        # exact name first, then section-prefixed copies ("TPC.TriageCompute.<metric>")
        for h in [m] + [h for h in head if h.endswith("." + m)]:
            if h not in col:
                continue
            i = col[h]
            try:
                res[key] = float(vals[i].replace(",", "")) * SCALE.get(units[i], 1)
                break
            except ValueError:
                continue
    if "duration" in res:
        res["duration_us"] = res.pop("duration") * 1e6
    if "dram_read" in res and "dram_write" in res:
        res["dram_bytes_per_launch"] = res["dram_read"] + res["dram_write"]
        res["dram_gbps"] = res["dram_bytes_per_launch"] / (res["duration_us"] * 1e-6) / 1e9
    return res


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    head = rows[0]
    ci = {h: i for i, h in enumerate(head)}
    per = {}
    for r in rows[1:]:
        if len(r) < len(head) or r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ci["Kernel Name"]]
        short = re.sub(r"\(.*", "", name)
        short = re.sub(r"^.*::", "", short)
        if any(k in short for k in SETUP_KERNELS):
            continue
        unit = r[ci["Metric Unit"]]
        t = float(r[ci["Metric Value"]].replace(",", "")) * SCALE.get(unit, 1)
        d = per.setdefault(short, [0, 0.0])
        d[0] += 1
        d[1] += t
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed+warmup+timing-pass steps in the captured bench run (per-step shares)")
    a = ap.parse_args()
    for rep in a.reports:
        s = summarise(rep)
        name = os.path.basename(rep).replace(".ncu-rep", "")
        if name.startswith(a.round + "_"):
            name = name[len(a.round) + 1:]
        with open(os.path.join(HERE, f"{a.round}_{name}.json"), "w") as f:
            json.dump(s, f, indent=1)
        if name == "c2_score_tc":
            with open(os.path.join(HERE, "ncu_C2_score_summary.json"), "w") as f:
                json.dump({"source": f"profiles/{a.round}_{name}.json", "kernel": s["kernel"],
                           "dram_bytes_per_launch": s.get("dram_bytes_per_launch"),
                           "duration_us": s.get("duration_us")}, f, indent=1)
        print(name, json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}))
    if a.launches:
        per = launches(a.launches)
        total = sum(v[1] for v in per.values())
        lines = [f"# {a.round}: ncu launch list of `bench.py` (C2), serialised, cold cache",
                 "", "Command: `ncu --metrics gpu__time_duration.sum --clock-control none python bench.py "
                 "--steps 2 --warmup 3 --no-cpu-baseline --no-e2e` (3 warm-up + 3 timing-pass + 2 timed "
                 "steps = 8 launches per kernel; data generation excluded).  Per-launch times are "
                 "serialised and cold-cache: compare shares, not absolute step time.", "",
                 "| kernel | launches | total µs | mean µs | share of step |", "|---|---|---|---|---|"]
        for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| {k} | {n} | {t * 1e6:.1f} | {t / n * 1e6:.2f} | {t / total:.1%} |")
        with open(os.path.join(HERE, f"{a.round}_launches_bench_C2.md"), "w") as f:
            f.write("\n".join(lines) + "\n")
        print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
