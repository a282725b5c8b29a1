"""Plan / wire-frame / checkpoint formats against reference golden bytes
(tests/golden/formats.json, config1_plan.txt from make_golden.py)."""

import json
import os

import numpy as np
import pytest

import paper_2401_01728_b200 as rv
from paper_2401_01728_b200 import formats
from conftest import GOLDEN


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "formats.json")) as f:
        return json.load(f)


def test_reads_reference_plan(golden):
    plan = formats.read_plan_file(os.path.join(GOLDEN, "config1_plan.txt"))
    assert [r.length for r in plan.schedule.rings] == golden["ring_lengths"] == [786688, 32896, 1290]
    assert plan.schedule.total_params == golden["total"] == 820874
    assert plan.cluster_ids == [1, 2]
    assert plan.node_of(2, 1) == "c2n1"
    # round trip of the [rings] section
    text = open(os.path.join(GOLDEN, "config1_plan.txt")).read()
    ours = formats.rings_section(plan.schedule)
    assert ours.strip() == text[text.index("[rings]"):].strip()
    # the builder from the spans gives the same schedule (clusterform.py:314)
    assert rv.build_ring_schedule(plan.layouts) == plan.schedule


def test_plan_schema_errors():
    with pytest.raises(rv.SchemaError):
        formats.read_plan("# schema: something-else\n[rings]\n")
    text = open(os.path.join(GOLDEN, "config1_plan.txt")).read()
    with pytest.raises(rv.LayoutError):
        formats.read_plan(text.replace("\n1 786688 32896 1:1,2:1", "\n1 786689 32896 1:1,2:1"))


def test_frames_golden(golden):
    for fr in golden["frames"]:
        b = formats.encode_frame(fr["kind"], fr["ring_id"], fr["round"], fr["offset"], np.array(fr["payload"]))
        assert b.hex() == fr["hex"]
        kind, rid, rnd, off, payload, used = formats.decode_frame(b + b"trailing")
        assert (kind, rid, rnd, off, used) == (fr["kind"], fr["ring_id"], fr["round"], fr["offset"], len(b))
        assert payload.tobytes() == np.array(fr["payload"], dtype="<f8").tobytes()
    with pytest.raises(rv.ProtocolError, match="truncated"):
        formats.decode_frame(formats.encode_frame("control", 0, 0, 0, np.zeros(2))[:10])
    with pytest.raises(rv.ProtocolError):
        formats.encode_frame("nonsense", 0, 0, 0, np.zeros(1))
    with pytest.raises(rv.ProtocolError):
        formats.decode_frame(b"\x01")


def test_owner_chunk_frames():
    sched = rv.build_ring_schedule({c: [rv.ParamRange(0, 10), rv.ParamRange(10, 5)] for c in range(3)})
    vals = np.arange(15.0)
    frames = formats.owner_chunk_frames(sched, vals, position=1, n_clusters=3)
    kinds = [formats.decode_frame(f) for f in frames]
    assert [(k[1], k[2], k[3]) for k in kinds] == [(0, 3, 4), (1, 3, 12)]
    np.testing.assert_array_equal(kinds[0][4], vals[4:7])
    np.testing.assert_array_equal(kinds[1][4], vals[12:14])


def test_checkpoint_golden(golden, tmp_path):
    p = tmp_path / "x.ckpt"
    formats.write_checkpoint(p, np.array([1.0, -2.5, 3e-300]))
    assert p.read_bytes().hex() == golden["checkpoint_hex"]
    np.testing.assert_array_equal(formats.read_checkpoint(p), [1.0, -2.5, 3e-300])
    p.write_bytes(b"NOTACKPT" + p.read_bytes()[8:])
    with pytest.raises(rv.SchemaError):
        formats.read_checkpoint(p)
