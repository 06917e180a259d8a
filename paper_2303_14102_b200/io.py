"""Dataset CSV ingest and report emission, host side of the GPU engine.

read_csv / read_csv_text follow the reference parser (csv.cpp:54-168, csv.hpp): one
point per row, features as finite numbers, one label column of any text; no quoting;
blank lines skipped; the label column by position (default last) or by header name;
header auto-detected (a first row whose feature cells are not all numbers); errors name
the 1-based physical line.  Labels are densified by first appearance -- the dense order
validate_and_densify gives -- and handed to the C ABI as int32 codes, the original
strings kept as cluster names.

write_report follows report_io.cpp:15-68: csv ("index,own_cluster,neighbour_cluster,a,b,s"
plus a "# summary:" line) or jsonl (one object per point plus a summary object), every
double with 17 significant digits (std::to_chars general, precision 17 == "%.17g").
"""
from __future__ import annotations

import io
import math
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, TextIO, Tuple, Union

import numpy as np

from .api import IoError, SilhouetteReport, ValidationError


@dataclass
class CsvSchema:
    delimiter: str = ","
    label_index: int = -1          # -1: last column; ignored when label_name is set
    label_name: str = ""           # by header name (requires a header)
    has_header: Optional[bool] = None  # None: auto-detect


@dataclass
class CsvDataset:
    X: np.ndarray                  # [n, d] float64 (the reference's Matrix, one point per row)
    labels: np.ndarray             # [n] int32 codes in first-appearance order (dense ids)
    cluster_names: List[str]       # dense id -> original label text


def _trim(s: str) -> str:
    return s.strip(" \t\r")


def _number(cell: str) -> Optional[float]:
    if not cell or cell != cell.strip():
        return None
    try:
        # from_chars grammar: no leading '+', no hex/inf spelled with underscores
        if cell[0] == "+" or "_" in cell:
            return None
        return float(cell)
    except ValueError:
        return None


def read_csv_text(text: str, schema: CsvSchema = CsvSchema(), name: str = "<string>") -> CsvDataset:
    lines: List[Tuple[int, str]] = []
    for no, raw in enumerate(text.split("\n"), start=1):
        if _trim(raw):
            lines.append((no, raw))
    if not lines:
        raise ValidationError(f"{name}: no data rows")

    def fail(line: int, what: str):
        raise ValidationError(f"{name}, line {line}: {what}")

    first = [_trim(c) for c in lines[0][1].split(schema.delimiter)]
    ncol = len(first)
    if ncol < 2:
        fail(lines[0][0], "need at least one feature column plus the label column")
    if schema.label_name:
        label_col = ncol
    else:
        idx = ncol + schema.label_index if schema.label_index < 0 else schema.label_index
        if idx < 0 or idx >= ncol:
            raise ValidationError(f"{name}: label column {schema.label_index} outside the {ncol} columns present")
        label_col = idx
    if schema.label_name:
        has_header = True
    elif schema.has_header is not None:
        has_header = schema.has_header
    else:
        has_header = any(_number(first[c]) is None for c in range(ncol) if c != label_col)
    if schema.label_name:
        if not has_header:
            raise ValidationError(f"{name}: label column by name requires a header row")
        if schema.label_name not in first:
            raise ValidationError(f"{name}: no header column named '{schema.label_name}'")
        label_col = first.index(schema.label_name)
    body = lines[1:] if has_header else lines
    if not body:
        raise ValidationError(f"{name}: no data rows")
    n, d = len(body), ncol - 1
    X = np.empty((n, d), np.float64)
    codes = np.empty(n, np.int32)
    names: List[str] = []
    index = {}
    for r, (no, raw) in enumerate(body):
        cells = [_trim(c) for c in raw.split(schema.delimiter)]
        if len(cells) != ncol:
            fail(no, f"expected {ncol} columns, got {len(cells)} (inconsistent dimensionality)")
        l = 0
        for c, cell in enumerate(cells):
            if c == label_col:
                continue
            v = _number(cell)
            if v is None:
                fail(no, f"cannot parse '{cell}' as a number")
            if not math.isfinite(v):
                fail(no, f"non-finite feature value '{cell}'")
            X[r, l] = v
            l += 1
        lab = cells[label_col]
        if not lab:
            fail(no, "empty label")
        if lab not in index:
            index[lab] = len(names)
            names.append(lab)
        codes[r] = index[lab]
    # read_csv_text ends in validate_and_densify (csv.cpp:158, dataset.cpp:29-57): the
    # dataset-level invariants come back from the reader itself, as in the reference.
    if n < 2:
        raise ValidationError(f"dataset needs at least 2 points, got {n}")
    if len(names) < 2:
        raise ValidationError(f"silhouette undefined for a single cluster: need K >= 2, got K = {len(names)}")
    return CsvDataset(X, codes, names)


def read_csv(path: Union[str, os.PathLike], schema: CsvSchema = CsvSchema()) -> CsvDataset:
    try:
        with open(path, "rb") as f:
            text = f.read().decode("utf-8")
    except OSError as e:
        raise IoError(f"cannot open '{os.fspath(path)}' for reading") from e
    return read_csv_text(text, schema, os.fspath(path))


def format_double17(v: float) -> str:
    """std::to_chars(general, 17) (report_io.cpp:15-20)."""
    return "%.17g" % float(v)


def write_points_csv(ds: CsvDataset, path: Union[str, os.PathLike]) -> None:
    """"f0,...,f{D-1},label" with 17-digit features; read_csv of it reproduces the data."""
    try:
        with open(path, "w", newline="") as out:
            out.write(",".join(f"f{l}" for l in range(ds.X.shape[1])) + ",label\n")
            for i in range(ds.X.shape[0]):
                out.write(",".join(format_double17(v) for v in ds.X[i]) + "," + ds.cluster_names[ds.labels[i]] + "\n")
    except OSError as e:
        raise IoError(f"cannot open '{os.fspath(path)}' for writing") from e


def _write(report: SilhouetteReport, out: TextIO, fmt: str, shards: int) -> None:
    own, nb = report.own, report.neighbour
    a = report.a if report.a is not None else np.zeros_like(report.s)
    b = report.b if report.b is not None else np.zeros_like(report.s)
    f = format_double17
    if fmt == "csv":
        out.write("index,own_cluster,neighbour_cluster,a,b,s\n")
        for i in range(report.s.shape[0]):
            out.write(f"{i},{own[i]},{nb[i]},{f(a[i])},{f(b[i])},{f(report.s[i])}\n")
        out.write(f"# summary: mean={f(report.mean)} metric={report.metric} engine={report.engine} "
                  f"shards={shards} wall_time_ms={f(report.wall_time_ms)}\n")
    elif fmt == "jsonl":
        for i in range(report.s.shape[0]):
            out.write(f'{{"index":{i},"own":{own[i]},"neighbour":{nb[i]},"a":{f(a[i])},'
                      f'"b":{f(b[i])},"s":{f(report.s[i])}}}\n')
        out.write(f'{{"mean":{f(report.mean)},"metric":"{report.metric}","engine":"{report.engine}",'
                  f'"shards":{shards},"wall_time_ms":{f(report.wall_time_ms)}}}\n')
    else:
        raise ValidationError(f"unknown format '{fmt}' (use csv or jsonl)")


def write_report(report: SilhouetteReport, dest: Union[str, os.PathLike, TextIO], fmt: str = "jsonl") -> None:
    """write_report (report_io.cpp:50-68) to a path or a text stream."""
    shards = getattr(report, "shards", 1)
    if hasattr(dest, "write"):
        _write(report, dest, fmt, shards)
        return
    try:
        with open(dest, "w", newline="") as out:
            _write(report, out, fmt, shards)
    except OSError as e:
        raise IoError(f"cannot open '{os.fspath(dest)}' for writing") from e


def report_text(report: SilhouetteReport, fmt: str = "jsonl") -> str:
    buf = io.StringIO()
    write_report(report, buf, fmt)
    return buf.getvalue()
