"""bench.py's JSON-line contract, CPU side: the reference arm (the CPU
restatement timed on host cores) prints one line with the driver's keys, and
the own arm refuses to run without a GPU instead of falling back to the CPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout,
                          env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})


@pytest.mark.timeout(600)
def test_reference_arm_prints_one_contract_line():
    p = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "samples/s" and d["higher_is_better"] is True
    assert d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]


@pytest.mark.timeout(300)
def test_own_arm_fails_without_gpu():
    p = _run("--steps", "1", "--warmup", "3", timeout=300)
    assert not [l for l in p.stdout.splitlines() if l.startswith("{")], p.stdout[-1000:]
    assert "CUDA" in p.stderr or "NVIDIA" in p.stderr or "cuda" in p.stderr


def test_b200_plan_report_picks_the_fastest_amp():
    sys.path.insert(0, ROOT)
    import bench
    for world in (2, 4, 8):
        r = bench.b200_plan_report(world)
        ok = [a for a in r["amps"] if "bp_predicted_us" in a]
        assert ok and r["bp_star_predicted_us"] == min(a["bp_predicted_us"] for a in ok)
        assert all(max(a["gpus_per_layer"]) <= world for a in ok)
        # overlapping the allreduce with the backward never predicts slower
        assert r["dp_overlapped_predicted_us"] <= r["dp_serial_predicted_us"]
    one = bench.b200_plan_report(1)
    assert one["dp_overlapped_predicted_us"] == pytest.approx(one["dp_serial_predicted_us"])


def test_host_timings_of_the_planner_and_simulator():
    sys.path.insert(0, ROOT)
    import bench
    h = bench.host_timings(8)
    assert 0 < h["plan_ms_median_of_20"] < 1000 and h["simulate_two_phase_bp_col_s"] > 0
