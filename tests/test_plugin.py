"""The drop-in seams: plugin.install() on the reference package, and the
drain-barrier controller's token protocol (CPU; the GPU cycle is replaced by
a stand-in so only host logic is exercised here -- GPU parity of the cycle
itself is in test_gpu_parity.py)."""

import heapq

import numpy as np
import pytest

import paper_2401_01728_b200 as rv
from paper_2401_01728_b200 import multiring as mr
from paper_2401_01728_b200 import plugin
from oracle import ring_oracle


def _oracle_mean(schedule, vals, acc="f64"):
    cids = sorted(vals)
    out = ring_oracle.ring_mean([r.start for r in schedule.rings], [r.length for r in schedule.rings],
                                [np.asarray(vals[c]) for c in cids])
    return dict(zip(cids, out))


class _Msg:
    def __init__(self, kind, sender, receiver, step_tag, payload=None, extra=None, **_):
        self.kind, self.sender, self.receiver, self.step_tag = kind, sender, receiver, step_tag
        self.payload, self.extra = payload, extra or {}


class _Net:
    """Minimal FIFO network with the reference Network's send/register shape."""

    Message = _Msg

    def __init__(self):
        self.q, self.seq, self.handlers, self.now = [], 0, {}, 0.0

    def register(self, name, fn):
        self.handlers[name] = fn

    def send(self, msg, now):
        heapq.heappush(self.q, (now + 1e-3, self.seq, msg))
        self.seq += 1

    def run(self):
        while self.q:
            t, _, msg = heapq.heappop(self.q)
            self.now = t
            self.handlers[msg.receiver](msg, t)


def test_controller_token_protocol(monkeypatch):
    import sys
    import types

    mod = types.ModuleType("fake_simnet")
    mod.Message = _Msg
    sys.modules["fake_simnet"] = mod
    _Net.__module__ = "fake_simnet"
    monkeypatch.setattr(mr, "apply_ring_mean", _oracle_mean)
    lay = {c: [rv.ParamRange(0, 5), rv.ParamRange(5, 7)] for c in (2, 9, 4)}
    sched = rv.build_ring_schedule(lay)
    rng = np.random.Generator(np.random.Philox(key=1))
    working = {c: rng.normal(size=12) for c in lay}
    want = _oracle_mean(sched, working)
    net = _Net()
    ctl = rv.AllReduceController(sched, working, net, rv.default_node_name)
    for ring in sched.rings:
        for m in ring.members:
            net.register(rv.default_node_name(*m), lambda msg, t: ctl.handle(msg, t))
    ctl.kickoff(0.0)
    assert not ctl.done()  # tokens in flight: the orchestrator's router will complete the cycle
    assert "token" in ctl.stall_report()
    net.run()
    assert ctl.done()
    assert ctl.stall_report() == "no ring is stalled"
    assert [s.rounds for s in ctl.stats()] == [4, 4]
    for c in lay:
        np.testing.assert_array_equal(working[c], want[c])
    with pytest.raises(rv.ProtocolError):
        ctl.handle(_Msg("ring_chunk", "a", "b", 0, extra={"ring": 0}), 0.0)


def test_install_patches_reference_seams():
    from conftest import import_reference

    ravnest = import_reference("ravnest")
    import ravnest.multiring as ref_mr
    import ravnest.orchestrator as ref_orch
    from ravnest.errors import ConfigError as RefConfig, StallError as RefStall

    orig = (ref_mr.apply_ring_mean, ref_mr.AllReduceController, ref_orch.AllReduceController)
    plugin.install(ravnest)
    try:
        assert ref_mr.apply_ring_mean is not orig[0]
        assert ref_orch.AllReduceController is ref_mr.AllReduceController
        assert issubclass(ref_orch.AllReduceController, rv.AllReduceController)
        # errors surface as the reference's own classes
        sched = ref_mr.build_ring_schedule({0: [ref_mr.ParamRange(0, 4)], 1: [ref_mr.ParamRange(0, 4)]})
        with pytest.raises(RefStall, match=r"ring=0, round=\d+, member=\(1, 0\)"):
            ref_mr.run_allreduce(sched, {0: np.ones(4), 1: np.ones(4)}, max_events=1)
        with pytest.raises(RefConfig):
            ref_mr.run_allreduce(sched, {0: np.ones(4)})
    finally:
        plugin.uninstall(ravnest)
    assert (ref_mr.apply_ring_mean, ref_mr.AllReduceController, ref_orch.AllReduceController) == orig
