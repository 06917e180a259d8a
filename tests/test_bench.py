"""bench.py host logic on CPU: the strong-scaling row partition is the reference's
plan_shards (engine.cpp:8-25, checked against the oracle's restatement), the default
workload is the largest single-GPU config with C4 beside it, and the roofline peaks come
from MEASURED_PEAKS.json."""
import sys

import pytest

import oracle

sys.argv = ["bench.py"]
import bench  # noqa: E402


@pytest.mark.parametrize("n,w", [(10, 3), (7, 8), (100_000_000, 8), (40_000_000, 3), (5, 1), (2, 2)])
def test_plan_shards_matches_reference(n, w):
    assert bench.plan_shards(n, w) == oracle.plan_shards(n, w)


def test_default_workload_is_c5_with_c4(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert a.config == "C5" and a.also == ["C4"] and a.gpus == 1
    monkeypatch.setattr(sys, "argv", ["bench.py", "--config", "C2"])
    assert bench.parse().also == []


def test_relaunch_only_outside_torchrun(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "1"])
    assert bench.maybe_relaunch(bench.parse()) is None
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    assert bench.maybe_relaunch(bench.parse()) is None


def test_peaks_and_cpu_sample_size():
    pk = bench.measured_peaks()
    assert pk["hbm"] > 1000 and pk["tc_sustained"] > 100
    rows = bench.cpu_sample_rows("C5", 768, 4096)
    assert 2 * 4096 <= rows <= 5_000_000
