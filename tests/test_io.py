"""Dataset CSV ingest and report emission (csv.cpp, report_io.cpp) and the
CLI's argument/error handling -- host-side, no GPU (the GPU run is in test_gpu_parity)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2303_14102_b200.api import IoError, SilhouetteReport, ValidationError
from paper_2303_14102_b200.io import (CsvDataset, CsvSchema, format_double17, read_csv, read_csv_text,
                                      report_text, write_points_csv)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_autodetect_and_first_appearance_labels():
    ds = read_csv_text("x,y,cls\n1,2,b\n\n3,4,a\n5,6,b\n")
    assert ds.X.tolist() == [[1, 2], [3, 4], [5, 6]]
    assert ds.labels.tolist() == [0, 1, 0] and ds.cluster_names == ["b", "a"]
    ds = read_csv_text("1,2,7\n3,4,9\n")  # no header: all feature cells numeric
    assert ds.X.shape == (2, 2) and ds.cluster_names == ["7", "9"]


def test_label_by_index_name_and_delimiter():
    ds = read_csv_text("lab;f0;f1\nq;1;2\nr;3;4\n", CsvSchema(delimiter=";", label_index=0))
    assert ds.X.tolist() == [[1, 2], [3, 4]] and ds.cluster_names == ["q", "r"]
    ds = read_csv_text("f0,who,f1\n1,u,2\n3,v,4\n", CsvSchema(label_name="who"))
    assert ds.X.tolist() == [[1, 2], [3, 4]] and ds.cluster_names == ["u", "v"]


@pytest.mark.parametrize("text,frag", [
    ("", "no data rows"),
    ("a,b\n", "no data rows"),
    ("1\n", "line 1: need at least one feature column"),
    ("1,2,a\n3,a\n", "line 2: expected 3 columns, got 2"),
    ("1,2,a\n3,zz,b\n", "line 2: cannot parse 'zz' as a number"),
    ("1,2,a\n3,inf,b\n", "line 2: non-finite feature value 'inf'"),
    ("1,2,a\n3,4, \n", "line 2: empty label"),
])
def test_csv_errors_name_the_line(text, frag):
    with pytest.raises(ValidationError, match=frag):
        read_csv_text(text)


def test_label_name_errors():
    with pytest.raises(ValidationError, match="no header column named 'nope'"):
        read_csv_text("a,b\n1,2\n", CsvSchema(label_name="nope"))
    with pytest.raises(ValidationError, match="outside the 2 columns"):
        read_csv_text("1,2\n", CsvSchema(label_index=5))


def test_points_csv_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    ds = CsvDataset(rng.normal(size=(40, 5)) * 1e3, rng.integers(0, 3, 40).astype(np.int32), ["p", "q", "r"])
    path = tmp_path / "pts.csv"
    write_points_csv(ds, path)
    back = read_csv(path)
    assert np.array_equal(back.X, ds.X)  # 17 significant digits: exact
    assert [back.cluster_names[c] for c in back.labels] == [ds.cluster_names[c] for c in ds.labels]


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(IoError):
        read_csv(tmp_path / "absent.csv")


def test_report_emission_formats():
    rep = SilhouetteReport(np.array([1 - 1 / 16.5]), np.array([1]), np.array([0]), np.array([1.0]),
                           np.array([16.5]), 0.1, "squared_euclidean", "fast", 1, 0.0, ["7", "3"])
    assert format_double17(0.1) == "0.10000000000000001"
    csv = report_text(rep, "csv").splitlines()
    assert csv[0] == "index,own_cluster,neighbour_cluster,a,b,s"
    assert csv[1] == "0,0,1,1,16.5,0.93939393939393945"
    assert csv[2].startswith("# summary: mean=0.10000000000000001 metric=squared_euclidean engine=fast shards=1")
    js = [json.loads(x) for x in report_text(rep, "jsonl").splitlines()]
    assert js[0] == {"index": 0, "own": 0, "neighbour": 1, "a": 1.0, "b": 16.5, "s": 1 - 1 / 16.5}
    assert js[1]["mean"] == 0.1 and js[1]["engine"] == "fast"


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2303_14102_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


def test_cli_exit_codes_for_io_and_validation(tmp_path):
    assert _cli("score", "--input", str(tmp_path / "absent.csv")).returncode == 1
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2,a\n3,x,b\n")
    r = _cli("score", "--input", str(bad))
    assert r.returncode == 2 and "line 2" in r.stderr
    good = tmp_path / "good.csv"
    good.write_text("1,2,a\n3,4,b\n")
    assert _cli("score", "--input", str(good), "--metric", "euclid").returncode == 2
    assert _cli("score", "--input", str(good), "--engine", "slow").returncode == 2
