"""Per-call kernel table from an ncu launch list of bench.py.

    python profiles/summarize_launches.py gpurun_out/launches_bench_C5.csv --round r02f

The list is the `ncu --metrics gpu__time_duration.sum --clock-control none` pass over
`python bench.py --steps 2 --warmup 1`.  Launches are split into library calls at every
densify_collect_kernel; a call is a C5 call if it runs the CTA-pair scoring kernel and a C4 call
if it runs thr_kernel.  Per class: mean time per kernel over the calls and its share of the call.
Times are serialised and cold-cache (and not power-capped like the bench's long steps): compare
shares, not absolutes.
"""
import argparse
import collections
import csv
import json
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))


def short(name):
    name = re.sub(r"\(.*$", "", name)  # drop the argument list
    name = name.replace("void ", "").replace("fsil::<unnamed>::", "").replace("tc::<unnamed>::", "")
    return name.replace("<unnamed>::", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--round", default="r02f")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    launches = [(short(r[ki]), float(r[vi].replace(",", "")) / 1e3) for r in rows[1:]]  # us
    # synthetic-data generation (datagen.cu) runs before the calls of a config: not part of a step
    setup = ("centres_kernel", "uniform_labels_kernel", "points_kernel", "nearest_kernel", "zipf_labels_kernel",
             "dirichlet_labels_kernel", "shuffle_kernel", "labels_kernel")
    launches = [(n, us) for n, us in launches if not n.startswith(setup)]
    calls, cur = [], None
    for name, us in launches:
        if name.startswith("densify_collect_kernel"):
            cur = []
            calls.append(cur)
        if cur is not None:
            cur.append((name, us))
    out = {"note": __doc__.split("\n\n")[2].replace("\n", " "), "source": os.path.basename(a.csv)}
    for cls, marker in (("C5", "score_tc_pair_kernel"), ("C4", "thr_kernel")):
        sel = [c for c in calls if any(n.startswith(marker) for n, _ in c)]
        if not sel:
            continue
        per = collections.OrderedDict()
        for c in sel:
            for n, us in c:
                per.setdefault(n, []).append(us)
        total = sum(sum(v) for v in per.values()) / len(sel)
        out[cls] = {"calls": len(sel), "launches_per_call": sum(len(c) for c in sel) / len(sel), "total_us": total,
                    "kernels": [{"kernel": n, "us": sum(v) / len(sel), "share": sum(v) / len(sel) / total}
                                for n, v in per.items()]}
    path = os.path.join(HERE, f"{a.round}_launches_bench.json")
    json.dump(out, open(path, "w"), indent=1)
    for cls in ("C5", "C4"):
        if cls in out:
            print(cls, f"{out[cls]['total_us'] / 1e3:.2f} ms per call, {out[cls]['launches_per_call']:.0f} launches")
            for k in out[cls]["kernels"]:
                print(f"  {k['us']:12.1f} us {k['share']:7.2%}  {k['kernel']}")


if __name__ == "__main__":
    main()
