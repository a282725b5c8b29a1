"""The drop-in at the reference's own seam, on the GPU.

The UNMODIFIED reference (baseline/_ref: the offline install that travels to
the GPU box; /root/reference in the dev container) trains twice per
scenario: plain, and with ``plugin.install(ravnest)`` routing both averaging
seams to this package -- ``multiring.apply_ring_mean`` for the snapshot
barrier (orchestrator.py:325-332) and ``AllReduceController`` for the drain
barrier (orchestrator.py:339-363).  Everything the reference reports must be
identical: final cluster parameters, averaging-cycle records (checkpoint
times included), the per-update metrics, the virtual clock and the network
trace (the drop-in controller replays the ring's messages with the chunks'
byte counts, multiring.py:185-225).
"""

import numpy as np
import pytest

from conftest import bits_equal, import_reference

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import c_oracle  # noqa: E402
from paper_2401_01728_b200 import multiring as mr  # noqa: E402
from paper_2401_01728_b200 import plugin  # noqa: E402

SCENARIOS = [
    # name, peers per cluster, MLP widths, barrier, kappa, k_target, link latency
    ("snapshot-2x3", [3, 3], [16, 24, 12, 4], "snapshot", 4, 72, 0.0),
    ("drain-2x3", [3, 3], [16, 24, 12, 4], "drain", 4, 72, 0.0),
    ("snapshot-nested-3/2/1/3", [3, 2, 1, 3], [12, 16, 16, 8], "snapshot", 5, 96, 0.0),
    ("drain-3x2-kappa1", [2, 2, 2], [8, 12, 6], "drain", 1, 30, 0.0),
    ("drain-nested-latency", [3, 2, 1, 3], [12, 16, 16, 8], "drain", 3, 72, 2e-3),
]


def make_plan(ravnest, peer_counts, arch, seed=3, batch_size=2):
    from ravnest import modelcore
    from ravnest.clusterform import ModelFootprint, plan_session
    from ravnest.simnet import NodeSpec

    model, params = modelcore.build_model(arch, seed, "tanh", "mse")
    fp = ModelFootprint.from_model(model, batch_size)
    pool, assignment = [], []
    for ci, count in enumerate(peer_counts, start=1):
        for j in range(count):
            pool.append(NodeSpec(f"c{ci}n{j}", fp.M, 1e9, 1.0))
            assignment.append(ci)
    return model, params, plan_session(pool, fp, len(peer_counts), model, assignment=assignment)


@pytest.mark.parametrize("name,peers,arch,mode,kappa,k_target,latency", SCENARIOS, ids=[s[0] for s in SCENARIOS])
def test_reference_train_identical_with_plugin(name, peers, arch, mode, kappa, k_target, latency):
    ravnest = import_reference("ravnest")
    from ravnest import data
    from ravnest.orchestrator import TrainConfig, train

    model, params, plan = make_plan(ravnest, peers, arch)
    dataset = data.make_dataset("mlp", model, 96, 5)
    cfg = TrainConfig(eta=0.05, kappa=kappa, k_target=k_target, batch_size=2, seed=7, barrier_mode=mode,
                      default_latency=latency, trace_enabled=True)
    ref = train(model, params.values, plan, cfg, dataset)
    calls = {"n": 0}
    real = mr._HostCycle.launch

    def counted(self, inputs):
        calls["n"] += 1
        return real(self, inputs)

    plugin.install(ravnest)
    try:
        mr._HostCycle.launch = counted
        gpu = train(model, params.values, plan, cfg, dataset)
    finally:
        mr._HostCycle.launch = real
        plugin.uninstall(ravnest)
    assert calls["n"] == ref.clock.cycle > 0  # every averaging cycle went through the GPU
    for cid in ref.cluster_values:
        assert bits_equal(gpu.cluster_values[cid], ref.cluster_values[cid]), cid
    assert bits_equal(gpu.mean_values, ref.mean_values)
    assert [(c.t, c.virtual_time, c.grad_norm, c.loss, c.spread) for c in gpu.checkpoints] == \
           [(c.t, c.virtual_time, c.grad_norm, c.loss, c.spread) for c in ref.checkpoints]
    assert gpu.metrics_hash() == ref.metrics_hash()  # includes the virtual time of every update
    assert gpu.virtual_time == ref.virtual_time
    assert gpu.net_trace_csv == ref.net_trace_csv
    assert gpu.final_loss == ref.final_loss


def test_drain_controller_is_asynchronous():
    """kickoff() returns while the GPU cycle is still in flight; the rounds
    play out over the caller's network, and done() lands the means in the
    caller's ``working`` dict -- bitwise the reference's apply_ring_mean."""
    ravnest = import_reference("ravnest")
    from ravnest.multiring import ParamRange, build_ring_schedule, default_node_name
    from ravnest.simnet import Network, NodeSpec

    c, n = 8, 1 << 24  # 8 clusters x 128 MB of float64
    lay = {cid: [ParamRange(0, n // 2), ParamRange(n // 2, n - n // 2)] for cid in range(c)}
    sched = build_ring_schedule(lay)
    rng = np.random.Generator(np.random.Philox(key=3))
    working = {cid: rng.normal(0, 1, n) for cid in range(c)}
    want = c_oracle.ring_mean([r.start for r in sched.rings], [r.length for r in sched.rings],
                              [working[cid] for cid in range(c)], threads=8)
    nodes = {default_node_name(*m): NodeSpec(default_node_name(*m), 1.0, 1e9) for r in sched.rings for m in r.members}
    net = Network(nodes, default_latency=1e-4)
    ctl = mr.AllReduceController(sched, working, net, default_node_name)
    for name in nodes:
        net.register(name, lambda msg, now: ctl.handle(msg, now))
    ctl.kickoff(0.0)
    in_flight = not ctl.gpu_ready()
    assert not ctl.done()  # no round has been delivered yet
    net.run_until(predicate=ctl.done, max_events=10_000)
    assert ctl.done()
    assert in_flight, "kickoff waited for the GPU cycle"
    assert [s.rounds for s in ctl.stats()] == [2 * (c - 1)] * 2
    for cid in range(c):
        assert bits_equal(working[cid], want[cid]), cid
    del ravnest


def test_numpy_dropin_input_forms():
    """apply_ring_mean's numpy path takes what the reference's np.array(x,
    dtype=float64) takes (multiring.py:309): float32 or float64 arrays,
    strided views, lists; returns new float64 arrays bitwise the reference;
    inputs untouched; one cluster returns float64 copies."""
    ravnest = import_reference("ravnest")
    from ravnest import multiring as ref_mr

    lay = {cid: [ref_mr.ParamRange(0, 700), ref_mr.ParamRange(700, 301)] for cid in (3, 1, 7)}
    sched = ref_mr.build_ring_schedule(lay)
    rng = np.random.Generator(np.random.Philox(key=21))
    base = {cid: rng.normal(0, 1, 2 * 1001) for cid in lay}
    forms = {
        3: base[3][::2].astype(np.float32),   # float32, strided
        1: base[1][:1001].copy(),             # float64
        7: list(base[7][1001:]),              # a list
    }
    keep = {c: np.array(v, copy=True) for c, v in forms.items()}
    want = ref_mr.apply_ring_mean(sched, forms)
    got = mr.apply_ring_mean(sched, forms)
    assert sorted(got) == sorted(want)
    for c in lay:
        assert got[c].dtype == np.float64 and got[c].shape == (1001,)
        assert bits_equal(got[c], want[c]), c
        assert bits_equal(np.asarray(forms[c], dtype=keep[c].dtype), keep[c])  # inputs untouched
    one = mr.apply_ring_mean(sched, {3: forms[3]})
    assert one[3].dtype == np.float64 and bits_equal(one[3], forms[3].astype(np.float64))
    del ravnest
