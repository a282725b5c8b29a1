"""NVLink-aware cost model: calibration against the committed B200 sweep and
the CLI front end (CPU only)."""

import json
import os

import pytest

import paper_2401_01728_b200 as rv
from paper_2401_01728_b200 import cli, cost
from conftest import ROOT, GOLDEN

SWEEP = os.path.join(ROOT, "profiles", "r02", "sweep_r02_n4.jsonl")


def rows():
    with open(SWEEP) as f:
        return [json.loads(l) for l in f if l.strip()]


def test_models_fit_measured_sweep():
    for proto, tol in (("pull", 0.06), ("push", 0.18)):
        model, err = cost.fit(rows(), proto)
        assert err < tol, proto
        assert 600e9 < model.beta_Bps < 720e9
        assert abs(model.beta_Bps - cost.CALIBRATED[proto].beta_Bps) / model.beta_Bps < 0.01
        big = [r for r in rows() if r["bytes_per_cluster"] >= 32 << 20]
        assert cost.fit(big, proto)[1] < 0.04


def test_model_shape_and_reference_contrast():
    lay = {c: [rv.ParamRange(0, 1 << 20), rv.ParamRange(1 << 20, 1 << 20)] for c in range(4)}
    sched = rv.build_ring_schedule(lay)
    rep = cost.allreduce_cost_nvlink(sched)
    # shared links: the cycle is the sum of ring shares plus the fixed cost
    assert rep.critical_seconds == pytest.approx(sum(r.seconds for r in rep.rings) + cost.CALIBRATED["pull"].alpha_s)
    ref = rv.allreduce_cost(sched, bandwidth=770e9, elem_bytes=4)
    assert ref.critical_ratio == pytest.approx(0.5)  # the reference's independent-link assumption
    assert rep.critical_ratio == 1.0


def test_cli_allreduce_bench(capsys):
    assert cli.main(["allreduce-bench", "--plan", os.path.join(GOLDEN, "config1_plan.txt")]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["clusters"] == 2 and out["rings"] == 3 and out["params"] == 820874
    assert out["b200_pull"]["cycle_s"] > 0
    assert cli.main(["rings", "--plan", os.path.join(GOLDEN, "config1_plan.txt")]) == 0
    assert "ring_id=2,start=819584,len=1290" in capsys.readouterr().out
