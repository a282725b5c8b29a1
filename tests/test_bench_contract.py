"""The bench.py JSON contract on CPU: the reference arm (the only leg that
runs without a GPU) prints one well-formed line."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                          "--warmup", "3", "--ref-sample-params", "200000"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["warmup"] >= 3 and d["steps"] == 3
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert d["metric"] == json.load(f)["metric"]


def test_reference_arm_runs_the_unmodified_reference_on_the_full_workload():
    """With baseline/_ref installed the arm times the unmodified
    ravnest.multiring.apply_ring_mean on the whole parameter set (here
    ResNet-50's rings at C=2 to stay quick), capping the step count to its
    time budget and saying so."""
    from conftest import reference_path

    import pytest

    if reference_path() is None:
        pytest.skip("reference not installed")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "resnet50", "--clusters", "2", "--steps", "50", "--warmup", "5", "--ref-budget-s", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    d = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    assert d["cpu_baseline"]["kind"] == "reference" and "FULL workload" in d["cpu_baseline"]["sample"]
    assert 1 <= d["steps"] <= d["steps_requested"] == 50
    assert d["config"]["clusters"] == 2 and d["ms_per_step"] > 0 and d["value"] > 0
