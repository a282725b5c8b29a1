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


class _OracleCycle:
    """CPU stand-in for the GPU cycle (_HostCycle) so only host logic runs."""

    def __init__(self, schedule, n):
        self.schedule = schedule

    def launch(self, arrays):
        return ring_oracle.ring_mean([r.start for r in self.schedule.rings], [r.length for r in self.schedule.rings],
                                     [np.asarray(a, dtype=np.float64) for a in arrays])

    def ready(self):
        return True

    def wait(self):
        pass


def test_controller_replays_the_ring_protocol(monkeypatch):
    import sys
    import types

    mod = types.ModuleType("fake_simnet")
    mod.Message = _Msg
    sys.modules["fake_simnet"] = mod
    _Net.__module__ = "fake_simnet"
    monkeypatch.setattr(mr, "_HostCycle", _OracleCycle)
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
    assert not ctl.done()  # rounds in flight: the orchestrator's router completes the cycle
    assert "(ring=0, round=0, member=(2, 0))" in ctl.stall_report()
    net.run()
    assert ctl.done()
    assert ctl.stall_report() == "no ring is stalled"
    assert [s.rounds for s in ctl.stats()] == [4, 4]
    assert [s.messages for s in ctl.stats()] == [12, 12]  # 2(C-1) rounds x C members
    for c in lay:
        np.testing.assert_array_equal(working[c], want[c])
    with pytest.raises(rv.ProtocolError):
        ctl.handle(_Msg("ring_chunk", "a", "b", 0, extra={"ring": 0, "to_pos": 0, "round": 7, "chunk": 0}), 0.0)


def test_controller_reproduces_reference_virtual_time_and_trace(monkeypatch):
    """Over the reference's own simnet Network (slow heterogeneous links,
    latency), the drop-in controller's message replay gives the SAME virtual
    completion time, the same trace (time, kind, sender, receiver, tag,
    bytes) and the same stats as the unmodified reference controller
    (multiring.py:154-247) -- only the arithmetic moved to the GPU."""
    from conftest import import_reference

    import_reference("ravnest")
    from ravnest.multiring import AllReduceController as RefCtl, default_node_name
    from ravnest.multiring import random_instance
    from ravnest.simnet import Network, NodeSpec

    monkeypatch.setattr(mr, "_HostCycle", _OracleCycle)
    for key in (55, 56, 57):
        rng = np.random.Generator(np.random.Philox(key=key))
        inst = random_instance(rng, 4, max_peers=3, max_dim=300)
        bw = {}
        for ring in inst.schedule.rings:
            for member in ring.members:
                bw[f"c{member[0]}.p{member[1]}"] = float(rng.uniform(1e4, 1e6))
        runs = []
        for cls in (RefCtl, rv.AllReduceController):
            net = Network({n: NodeSpec(n, 1.0, b) for n, b in bw.items()}, default_latency=0.003)
            holder = {}
            for name in bw:
                net.register(name, lambda msg, now: holder["ctl"].handle(msg, now))
            working = {c: v.copy() for c, v in inst.cluster_values.items()}
            ctl = cls(inst.schedule, working, net, default_node_name)
            holder["ctl"] = ctl
            ctl.kickoff(0.0)
            net.run_until(predicate=ctl.done, max_events=100_000)
            assert ctl.done()
            runs.append((net.now, list(net.trace), [(s.ring_id, s.rounds, s.messages) for s in ctl.stats()], working))
        (t_ref, tr_ref, st_ref, w_ref), (t_ours, tr_ours, st_ours, w_ours) = runs
        assert t_ours == t_ref and t_ref > 0.003
        assert tr_ours == tr_ref
        assert st_ours == st_ref
        for c in w_ref:
            assert np.array_equal(w_ours[c], w_ref[c])


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


@pytest.mark.parametrize("mode,latency", [("snapshot", 0.0), ("drain", 0.0), ("drain", 2e-3)])
def test_reference_train_through_the_seam_host_logic(monkeypatch, mode, latency):
    """The reference's own train() with plugin.install, the GPU cycle
    replaced by the oracle (host logic only; tests/test_reference_seam_gpu.py
    runs the same on the GPU): parameters, checkpoints, metrics, virtual
    clock and network trace identical to the plain reference."""
    from conftest import import_reference

    ravnest = import_reference("ravnest")
    from ravnest import data, modelcore
    from ravnest.clusterform import ModelFootprint, plan_session
    from ravnest.orchestrator import TrainConfig, train
    from ravnest.simnet import NodeSpec

    model, params = modelcore.build_model([12, 16, 16, 8], 3, "tanh", "mse")
    fp = ModelFootprint.from_model(model, 2)
    pool, assignment = [], []
    for ci, count in enumerate([3, 2, 1, 3], start=1):
        for j in range(count):
            pool.append(NodeSpec(f"c{ci}n{j}", fp.M, 1e9, 1.0))
            assignment.append(ci)
    plan = plan_session(pool, fp, 4, model, assignment=assignment)
    dataset = data.make_dataset("mlp", model, 96, 5)
    cfg = TrainConfig(eta=0.05, kappa=3, k_target=72, batch_size=2, seed=7, barrier_mode=mode,
                      default_latency=latency, trace_enabled=True)
    ref = train(model, params.values, plan, cfg, dataset)
    monkeypatch.setattr(mr, "_HostCycle", _OracleCycle)
    plugin.install(ravnest)
    try:
        ours = train(model, params.values, plan, cfg, dataset)
    finally:
        plugin.uninstall(ravnest)
    for cid in ref.cluster_values:
        assert np.array_equal(ours.cluster_values[cid], ref.cluster_values[cid])
    assert [(c.t, c.virtual_time, c.loss) for c in ours.checkpoints] == [(c.t, c.virtual_time, c.loss) for c in ref.checkpoints]
    assert ours.metrics_hash() == ref.metrics_hash()
    assert ours.virtual_time == ref.virtual_time
    assert ours.net_trace_csv == ref.net_trace_csv
