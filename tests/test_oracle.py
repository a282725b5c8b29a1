"""Pin the CPU oracle (oracle/) to the unmodified reference's outputs.

Fixtures: tests/golden/ring_instances.npz (made by tests/golden/make_golden.py
from /root/reference).  Everything here is CPU-only.
"""

import numpy as np
import pytest

from conftest import bits_equal
from oracle import c_oracle, ring_oracle


def _rows(a):
    return [a[i] for i in range(a.shape[0])]


def test_fixture_sanity(golden_instances):
    assert len(golden_instances) >= 50
    assert {g.c for g in golden_instances} >= {2, 3, 4, 5, 6, 7, 8}
    # the reference's own invariant: event path == synchronous path bitwise
    for g in golden_instances:
        if g.run_allreduce is not None:
            assert bits_equal(g.run_allreduce, g.apply_ring_mean), g.name
            assert (g.rounds == 2 * (g.c - 1)).all()
            assert (g.messages == 2 * (g.c - 1) * g.c).all()


def test_numpy_closed_form_is_bitwise_reference(golden_instances):
    for g in golden_instances:
        got = ring_oracle.ring_mean(g.starts, g.lens, _rows(g.x), acc=ring_oracle.ACC_F64)
        assert bits_equal(np.stack(got), g.apply_ring_mean), g.name


def test_numpy_closed_form_f32_inputs_is_bitwise_reference(golden_instances):
    for g in golden_instances:
        got = ring_oracle.ring_mean(g.starts, g.lens, _rows(g.x32), acc=ring_oracle.ACC_F64)
        assert bits_equal(np.stack(got), g.apply_ring_mean_f32in), g.name


def test_round_simulation_is_bitwise_reference(golden_instances):
    for g in golden_instances:
        got = ring_oracle.ring_mean_rounds(g.starts, g.lens, _rows(g.x), dtype=np.float64)
        assert bits_equal(np.stack(got), g.apply_ring_mean), g.name


def test_fp32_ring_order_closed_form_equals_round_simulation(golden_instances):
    # the fp32 ring-order oracle: closed form vs message-order simulation in fp32
    for g in golden_instances:
        a = ring_oracle.ring_mean(g.starts, g.lens, _rows(g.x32), acc=ring_oracle.ACC_NATIVE)
        b = ring_oracle.ring_mean_rounds(g.starts, g.lens, _rows(g.x32), dtype=np.float32)
        assert bits_equal(np.stack(a), np.stack(b)), g.name


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_c_oracle_is_bitwise_reference(golden_instances, threads):
    for g in golden_instances:
        got = c_oracle.ring_mean(g.starts, g.lens, _rows(g.x), mode=c_oracle.MODE_F64, threads=threads)
        assert bits_equal(np.stack(got), g.apply_ring_mean), g.name
        got = c_oracle.ring_mean(g.starts, g.lens, _rows(g.x32), mode=c_oracle.MODE_F32_ACC64,
                                 threads=threads)
        assert bits_equal(np.stack(got), g.apply_ring_mean_f32in), g.name
        got = c_oracle.ring_mean(g.starts, g.lens, _rows(g.x32), mode=c_oracle.MODE_F32_NATIVE,
                                 threads=threads)
        want = ring_oracle.ring_mean(g.starts, g.lens, _rows(g.x32), acc=ring_oracle.ACC_NATIVE)
        assert bits_equal(np.stack(got), np.stack(want)), g.name


def test_c_oracle_f32_out_is_rounded_reference(golden_instances):
    for g in golden_instances:
        ins = [np.ascontiguousarray(r) for r in _rows(g.x32)]
        outs32 = [np.empty_like(r) for r in ins]
        c_oracle.ring_mean_into(c_oracle.MODE_F32_ACC64, g.starts, g.lens, ins, None, outs32, threads=2)
        with np.errstate(over="ignore"):
            want = g.apply_ring_mean_f32in.astype(np.float32)
        assert bits_equal(np.stack(outs32), want), g.name


def test_mean_reference_kats():
    # oracle.py KATs (test_oracle.py:31-38)
    v = np.arange(5.0)
    np.testing.assert_array_equal(ring_oracle.mean_reference([v, v, v]), v)
    got = ring_oracle.mean_reference([np.array([2.0, 4.0]), np.array([4.0, 8.0])])
    np.testing.assert_array_equal(got, [3.0, 6.0])


def test_reference_tolerance_contract(golden_instances):
    # criterion 1: ring mean vs scalar mean within 1e-12 on the floor-1 metric
    for g in golden_instances:
        if not g.name.startswith(("crit1", "kat_four", "wide")):
            continue
        want = ring_oracle.mean_reference(_rows(g.x))
        for row in g.apply_ring_mean:
            assert ring_oracle.floor1_rel_err(row, want) <= 1e-12, g.name


def test_chunk_bounds_kats(schedule_kats):
    for case in schedule_kats["chunk_bounds"]:
        got = ring_oracle.chunk_bounds(*case["args"])
        assert [list(b) for b in got] == case["bounds"]


def test_blend_identity_and_signed_zero():
    snap = np.array([1.0, -0.0, 2.5, 3.0], dtype=np.float32)
    live = snap.copy()
    mean = np.array([0.5, 0.0, -0.0, 1.0], dtype=np.float32)
    out = ring_oracle.blend(mean, live, snap)
    assert bits_equal(out, mean)
    live2 = snap - np.float32(0.25)
    out2 = ring_oracle.blend(mean, live2, snap)
    np.testing.assert_array_equal(out2, mean + (live2 - snap))
