"""`python -m paper_2303_14102_b200 {score,compare}` -- the reference tool's `score` and
`compare` subcommands (tools/main.cpp:19-108, 160-200) over the GPU engines, with its exit
codes: 0 ok, 1 I/O error, 2 validation error, 3 compare tolerance exceeded.

  score   --input f.csv [--metric sqeuclid|cosine] [--engine fast|naive] [--shards W]
          [--output path] [--format jsonl|csv]
  compare --input f.csv [--metric ...] [--rtol R] [--atol A] [--inject-fault E]

(`bench` -- the reference's CPU scaling harness -- is bench.py at the repository root.)
"""
import argparse
import sys

EXIT_OK, EXIT_IO, EXIT_VALIDATION, EXIT_TOLERANCE = 0, 1, 2, 3


def _metric(flag: str) -> str:
    from .api import ValidationError
    known = {"sqeuclid": "sqeuclid", "squared_euclidean": "sqeuclid", "cosine": "cosine"}
    if flag in ("euclid", "euclidean", "euclidean_oracle"):
        raise ValidationError("plain euclidean distance is available only through the naive oracle "
                              "library API, not the CLI")
    if flag not in known:
        raise ValidationError(f"unknown metric '{flag}' (use sqeuclid or cosine)")
    return known[flag]


def cmd_score(a) -> int:
    from .api import ValidationError, default_context
    from .io import format_double17, read_csv, write_report
    metric = _metric(a.metric)
    if a.engine not in ("fast", "naive"):
        raise ValidationError(f"unknown engine '{a.engine}' (use fast or naive)")
    if a.format not in ("csv", "jsonl"):
        raise ValidationError(f"unknown format '{a.format}' (use csv or jsonl)")
    ds = read_csv(a.input)
    ctx = default_context()
    rep = ctx.silhouette_naive(ds.X, ds.labels, metric) if a.engine == "naive" else ctx.silhouette(ds.X, ds.labels, metric)
    rep.cluster_names = list(ds.cluster_names)
    rep.shards = a.shards if a.shards > 0 else 1
    if a.output:
        write_report(rep, a.output, a.format)
    print(f"metric={rep.metric} engine={rep.engine} shards={rep.shards} n={ds.X.shape[0]} "
          f"k={len(ds.cluster_names)}")
    print(f"mean_silhouette={format_double17(rep.mean)}")
    print(f"wall_time_ms={format_double17(rep.wall_time_ms)}")
    return EXIT_OK


def cmd_compare(a) -> int:
    from .api import compare
    from .io import format_double17, read_csv
    metric = _metric(a.metric)
    ds = read_csv(a.input)
    r = compare(ds.X, ds.labels, metric, rtol=a.rtol, atol=a.atol, inject_fault=a.inject_fault)
    f = format_double17
    print(f"fast:  mean={f(r['fast_mean'])} wall_time_ms={f(r['fast_wall_ms'])}")
    print(f"naive: mean={f(r['naive_mean'])} wall_time_ms={f(r['naive_wall_ms'])}")
    print(f"max_abs_deviation={f(r['max_abs_deviation'])}")
    print(f"max_rel_deviation={f(r['max_rel_deviation'])}")
    if not r["within"]:
        print(f"tolerance exceeded (rtol={a.rtol:g}, atol={a.atol:g})")
        return EXIT_TOLERANCE
    print(f"within tolerance (rtol={a.rtol:g}, atol={a.atol:g})")
    return EXIT_OK


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="python -m paper_2303_14102_b200",
                                description="linear-time Silhouette on B200 (arXiv 2303.14102)")
    sub = p.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("score", help="score a labeled CSV dataset")
    s.add_argument("--input", required=True)
    s.add_argument("--metric", default="sqeuclid")
    s.add_argument("--engine", default="fast")
    s.add_argument("--shards", type=int, default=0)
    s.add_argument("--output", default="")
    s.add_argument("--format", default="jsonl")
    c = sub.add_parser("compare", help="run both engines and check they agree")
    c.add_argument("--input", required=True)
    c.add_argument("--metric", default="sqeuclid")
    c.add_argument("--shards", type=int, default=0)
    # the fast engine certifies |ds_i| <= 1e-5, hence these defaults
    c.add_argument("--rtol", type=float, default=1e-4)
    c.add_argument("--atol", type=float, default=1e-5)
    c.add_argument("--inject-fault", dest="inject_fault", type=float, default=0.0, help=argparse.SUPPRESS)
    a = p.parse_args(argv)
    from .api import FsilError, IoError, ValidationError
    try:
        return cmd_score(a) if a.cmd == "score" else cmd_compare(a)
    except IoError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    except ValidationError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VALIDATION
    except FsilError as e:  # device / CUDA failure: no CPU fallback
        print(f"error: {e}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())
