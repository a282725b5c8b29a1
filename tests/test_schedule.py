"""Host mirror of the schedule builders vs golden output of the reference
(tests/golden/schedule_kats.json, made from multiring.py:56-144,340-394),
plus the reference's own schedule unit tests (test_multiring.py:35-97,221-245)."""

import numpy as np
import pytest

import paper_2401_01728_b200 as rv
from paper_2401_01728_b200.multiring import _ideal_network_progress, _stall_text


def layouts_from_sizes(sizes):
    out = {}
    for cid, ss in sizes.items():
        start, lay = 0, []
        for s in ss:
            lay.append(rv.ParamRange(start, s))
            start += s
        out[int(cid)] = lay
    return out


def test_golden_schedules(schedule_kats):
    n_err = 0
    for case in schedule_kats["schedules"]:
        lay = layouts_from_sizes(case["sizes"])
        if "error" in case:
            n_err += 1
            with pytest.raises(getattr(rv, case["error"])) as ei:
                s = rv.build_ring_schedule(lay)
                rv.validate_schedule(s, lay)
            assert str(ei.value) == case["message"]
        else:
            s = rv.build_ring_schedule(lay)
            rv.validate_schedule(s, lay)
            assert s.dump() == case["dump"]
            assert s.total_params == case["total"]
    assert n_err >= 2


def test_golden_chunk_bounds(schedule_kats):
    for case in schedule_kats["chunk_bounds"]:
        assert [list(b) for b in rv.chunk_bounds(*case["args"])] == case["bounds"]


def test_golden_cost(schedule_kats):
    for case in schedule_kats["cost"]:
        s = rv.build_ring_schedule(layouts_from_sizes(case["sizes"]))
        rep = rv.allreduce_cost(s, bandwidth=case["bandwidth"], latency=case["latency"])
        got = [[r.ring_id, r.rounds, r.seg_bytes, r.bytes_per_member, r.seconds] for r in rep.rings]
        assert got == case["rings"]
        assert rep.critical_seconds == case["critical"]
        assert rep.single_ring_seconds == case["single"]


def test_reference_unit_cases():
    # test_multiring.py:36-74
    s = rv.build_ring_schedule(layouts_from_sizes({0: [10, 6], 1: [10, 6]}))
    assert s.rings[0].members == ((0, 0), (1, 0)) and s.rings[1].members == ((0, 1), (1, 1))
    s = rv.build_ring_schedule(layouts_from_sizes({0: [8, 8], 1: [16]}))
    assert s.rings[1].members == ((0, 1), (1, 0))
    lines = s.dump().splitlines()
    assert lines[0] == "# schema: ravnest-rings-v1"
    assert lines[1] == "ring_id=0,start=0,len=8,members=[(0,0),(1,0)]"
    assert lines[2] == "ring_id=1,start=8,len=8,members=[(0,1),(1,0)]"
    with pytest.raises(rv.LayoutError, match="different totals"):
        rv.build_ring_schedule(layouts_from_sizes({0: [10], 1: [12]}))
    with pytest.raises(rv.LayoutError, match="nest"):
        rv.build_ring_schedule(layouts_from_sizes({0: [4, 8], 1: [8, 4]}))
    with pytest.raises(rv.LayoutError):
        rv.build_ring_schedule({})


def test_cost_properties():
    # test_multiring.py:221-245 and acceptance criterion 8 (test_acceptance.py:241-268)
    rng = np.random.Generator(np.random.Philox(key=99))
    for _ in range(50):
        c = int(rng.integers(2, 8))
        sb = float(rng.integers(8, 10**7))
        assert rv.bytes_per_member(c, sb) == 2.0 * (c - 1) * sb / c
    for rings in (2, 3, 5):
        lay = {cid: [rv.ParamRange(r * 128, 128) for r in range(rings)] for cid in range(3)}
        rep = rv.allreduce_cost(rv.build_ring_schedule(lay), bandwidth=1e7)
        assert abs(rep.critical_ratio - 1.0 / rings) <= 1e-12
    rep = rv.allreduce_cost(rv.build_ring_schedule(layouts_from_sizes({c: [30] for c in range(3)})), bandwidth=1e6)
    assert rep.rings[0].rounds == 4


def test_run_allreduce_errors_without_gpu():
    s = rv.build_ring_schedule(layouts_from_sizes({0: [4]}))
    with pytest.raises(rv.ConfigError):
        rv.run_allreduce(s, {0: np.ones(4)})
    s = rv.build_ring_schedule(layouts_from_sizes({0: [4], 1: [4]}))
    with pytest.raises(rv.LayoutError):
        rv.run_allreduce(s, {0: np.ones(4), 1: np.ones(5)})
    # test_multiring.py:159-163: an event budget too small for the cycle
    with pytest.raises(rv.StallError, match=r"ring=0, round=\d+, member=\(1, 0\)"):
        rv.run_allreduce(s, {0: np.ones(4), 1: np.ones(4)}, max_events=1)


def test_stall_report_matches_reference_fifo():
    # same (ring, round, member) set the reference reports for every budget
    from conftest import import_reference

    ref = import_reference("ravnest.multiring")
    RefStall = import_reference("ravnest.errors").StallError

    rng = np.random.Generator(np.random.Philox(key=3))
    for _ in range(12):
        c = int(rng.integers(2, 6))
        inst = ref.random_instance(rng, c, max_peers=3, max_dim=40)
        sched = rv.build_ring_schedule(inst.layouts)
        needed = sum(2 * (c - 1) * c for _ in sched.rings)
        for budget in sorted({1, 2, 3, c + 1, needed // 3, needed // 2, needed - 1}):
            with pytest.raises(RefStall) as ei:
                ref.run_allreduce(inst.schedule, inst.cluster_values, max_events=budget)
            ref_report = str(ei.value).split("waiting on: ")[-1]
            ours = _stall_text(sched, _ideal_network_progress(sched, c, budget), c).split("waiting on: ")[-1]
            assert ours == ref_report


def test_builder_agrees_with_reference_on_random_layouts():
    """2000 random layouts (nested or not, zero-length submodels and rings,
    mismatched totals, gaps): same dump or the same exception class and
    message as the unmodified reference builder (multiring.py:56-105)."""
    import random

    from conftest import import_reference

    import_reference("ravnest")
    import ravnest.multiring as R

    rng = random.Random(1)
    for _ in range(2000):
        total = rng.randint(0, 12)
        lay = {}
        for c in range(rng.randint(1, 4)):
            pts = [0, *sorted(rng.choices(range(total + 1), k=rng.randint(0, 3))), total]
            lay[c * 3 + rng.randint(0, 2)] = [(pts[i], pts[i + 1] - pts[i]) for i in range(len(pts) - 1)]
        if rng.random() < 0.1:
            k = rng.choice(list(lay))
            lay[k] = lay[k][:-1] if len(lay[k]) > 1 else [(1, 2)]
        outcome = []
        for mod in (R, rv):
            try:
                outcome.append(mod.build_ring_schedule({c: [mod.ParamRange(a, b) for a, b in v]
                                                        for c, v in lay.items()}).dump())
            except Exception as e:  # noqa: BLE001 - compare class names and messages
                outcome.append((type(e).__name__, str(e)))
        assert outcome[0] == outcome[1], lay
