"""End-to-end drop-in check against the reference's own training loop.

Runs the UNMODIFIED reference (installed once into git-ignored baseline/_ref
with `pip install --no-deps --target baseline/_ref`) twice per scenario:
plain, and with `paper_2401_01728_b200.plugin.install(ravnest)` routing its
averaging seams (multiring.apply_ring_mean for the snapshot barrier,
AllReduceController for the drain barrier, orchestrator.py:320-363) to the
GPU.  Final cluster parameters, the averaging-cycle records and the metrics
must be bitwise identical.  Prints one JSON line.  Not part of the pytest
suite (the reference does not travel with the tests); run on a GPU box:

    python tools/integration_reference.py
"""

import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

import ravnest  # noqa: E402
from ravnest import data, modelcore  # noqa: E402
from ravnest.clusterform import ModelFootprint, plan_session  # noqa: E402
from ravnest.orchestrator import TrainConfig, train  # noqa: E402
from ravnest.simnet import NodeSpec  # noqa: E402

from paper_2401_01728_b200 import plugin  # noqa: E402


def make_plan(peer_counts, arch, seed=3, batch_size=2):
    model, params = modelcore.build_model(arch, seed, "tanh", "mse")
    fp = ModelFootprint.from_model(model, batch_size)
    pool, assignment = [], []
    for ci, count in enumerate(peer_counts, start=1):
        for j in range(count):
            pool.append(NodeSpec(f"c{ci}n{j}", fp.M, 1e9, 1.0))
            assignment.append(ci)
    return model, params, plan_session(pool, fp, len(peer_counts), model, assignment=assignment)


def digest(result) -> str:
    h = hashlib.sha256()
    for cid in sorted(result.cluster_values):
        h.update(np.ascontiguousarray(result.cluster_values[cid], dtype="<f8").tobytes())
    for ck in result.checkpoints:
        h.update(repr((ck.t, ck.grad_norm, ck.loss, ck.spread)).encode())
    return h.hexdigest()


def main():
    scenarios = [
        ("snapshot, 2 clusters x 3 peers, kappa 4", [3, 3], [16, 24, 12, 4], "snapshot", 4, 72),
        ("drain, 2 clusters x 3 peers, kappa 4", [3, 3], [16, 24, 12, 4], "drain", 4, 72),
        ("snapshot, 4 clusters, nested 3/2/1/3 peers", [3, 2, 1, 3], [12, 16, 16, 8], "snapshot", 5, 96),
        ("drain, 3 clusters, kappa 1", [2, 2, 2], [8, 12, 6], "drain", 1, 30),
    ]
    out = []
    ok = True
    for name, peers, arch, mode, kappa, k_target in scenarios:
        model, params, plan = make_plan(peers, arch)
        dataset = data.make_dataset("mlp", model, 96, 5)
        cfg = TrainConfig(eta=0.05, kappa=kappa, k_target=k_target, batch_size=2, seed=7, barrier_mode=mode)
        ref = train(model, params.values, plan, cfg, dataset)
        plugin.install(ravnest)
        try:
            gpu = train(model, params.values, plan, cfg, dataset)
        finally:
            plugin.uninstall(ravnest)
        same = digest(ref) == digest(gpu)
        # per-update metrics without the virtual-time column: the drain
        # barrier's ring messages occupy simulated link time in the reference,
        # the GPU cycle's zero-byte tokens do not
        strip = lambda r: [(m.t, m.cluster, m.peer, m.tau, m.loss, m.grad_norm) for m in r.metrics]
        same_metrics = strip(ref) == strip(gpu)
        ok &= same and same_metrics
        out.append({"scenario": name, "cycles": ref.clock.cycle, "rings": len(plan.ring_schedule.rings),
                    "params_and_cycles_bitwise_identical": same, "metrics_identical": same_metrics,
                    "digest": digest(ref)[:16]})
    print(json.dumps({"integration": "reference train() with plugin.install vs plain", "ok": ok,
                      "scenarios": out}))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
