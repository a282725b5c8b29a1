"""Generate golden fixtures from the UNMODIFIED reference (run in the dev container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ravnest from /root/reference/pkg/src (read-only; never needed at test
time) and records, for seeded inputs, exactly what the reference's averaging
path returns:

* ``ring_instances.npz`` -- per instance: ring starts/lengths, the C input
  vectors (float64), ``apply_ring_mean`` output (multiring.py:302-333),
  ``run_allreduce`` output (multiring.py:254-299) and the reference applied to
  the same inputs rounded to float32 (the fp32 product path's parity target).
  Instances come from ``multiring.random_instance`` (multiring.py:440-465)
  with the reference tests' own Philox keys (test_multiring.py:117-218,
  test_acceptance.py:28-51) plus edge cases (zero-length chunks, C up to 8,
  signed zeros, subnormals, infinities).
* ``schedule_kats.json`` -- ``build_ring_schedule`` dumps and error classes
  (multiring.py:56-131), ``chunk_bounds`` (:134-144), ``RingStats``
  (:234-238), ``bytes_per_member``/``allreduce_cost`` (:340-394).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from ravnest import multiring  # noqa: E402
from ravnest.errors import RavnestError  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def layouts_from_sizes(sizes_by_cluster):
    out = {}
    for cid, sizes in sizes_by_cluster.items():
        start, ranges = 0, []
        for s in sizes:
            ranges.append(multiring.ParamRange(start, s))
            start += s
        out[cid] = ranges
    return out


def record(store, name, schedule, values):
    cids = sorted(values)
    x = np.stack([np.asarray(values[c], dtype=np.float64) for c in cids]) if cids else None
    arm = multiring.apply_ring_mean(schedule, values)
    store[f"{name}/starts"] = np.array([r.start for r in schedule.rings], dtype=np.int64)
    store[f"{name}/lens"] = np.array([r.length for r in schedule.rings], dtype=np.int64)
    store[f"{name}/cids"] = np.array(cids, dtype=np.int64)
    store[f"{name}/x"] = x
    store[f"{name}/apply_ring_mean"] = np.stack([arm[c] for c in cids])
    if len(cids) >= 2:
        ev, stats = multiring.run_allreduce(schedule, values)
        store[f"{name}/run_allreduce"] = np.stack([ev[c] for c in cids])
        store[f"{name}/rounds"] = np.array([s.rounds for s in stats], dtype=np.int64)
        store[f"{name}/messages"] = np.array([s.messages for s in stats], dtype=np.int64)
    x32 = {c: np.asarray(values[c], dtype=np.float32) for c in cids}
    arm32 = multiring.apply_ring_mean(schedule, x32)
    store[f"{name}/x32"] = np.stack([x32[c] for c in cids])
    store[f"{name}/apply_ring_mean_f32in"] = np.stack([arm32[c] for c in cids])


def main():
    store: dict[str, np.ndarray] = {}
    names = []

    def add(name, schedule, values):
        record(store, name, schedule, values)
        names.append(name)

    # --- KATs straight from test_multiring.py -------------------------------
    sched = multiring.build_ring_schedule(layouts_from_sizes({0: [2], 1: [2]}))
    add("kat_two_cluster", sched, {0: np.array([2.0, 4.0]), 1: np.array([4.0, 8.0])})
    sched = multiring.build_ring_schedule(layouts_from_sizes({0: [6], 1: [6]}))
    add("kat_fixed_point", sched, {0: np.arange(6.0), 1: np.arange(6.0)})
    rng = np.random.Generator(np.random.Philox(key=5))
    sched = multiring.build_ring_schedule(layouts_from_sizes({c: [32, 16, 16] for c in range(4)}))
    add("kat_four_clusters_key5", sched, {c: rng.normal(0, 5, 64) for c in range(4)})
    for key, c, mp, md in ((31, 4, 3, 200), (55, 4, 3, 300)):
        inst = multiring.random_instance(np.random.Generator(np.random.Philox(key=key)), c,
                                         max_peers=mp, max_dim=md)
        add(f"kat_random_key{key}", inst.schedule, inst.cluster_values)
    rng = np.random.Generator(np.random.Philox(key=9))
    sched = multiring.build_ring_schedule(layouts_from_sizes({c: [20] for c in range(3)}))
    add("kat_idempotent_key9", sched, {c: rng.normal(size=20) for c in range(3)})

    # --- acceptance criterion 1 stream (test_acceptance.py:28-51), first 40 --
    rng = np.random.Generator(np.random.Philox(key=777))
    for i in range(40):
        c = int(rng.integers(2, 7))
        inst = multiring.random_instance(rng, c, max_peers=4, max_dim=4096)
        add(f"crit1_{i:02d}", inst.schedule, inst.cluster_values)

    # --- wider C (one cluster per GPU up to 8) and non-contiguous cluster ids
    rng = np.random.Generator(np.random.Philox(key=20241018))
    for i, c in enumerate((7, 8, 8, 5, 3, 2)):
        inst = multiring.random_instance(rng, c, max_peers=4, max_dim=3000)
        add(f"wide_c{c}_{i}", inst.schedule, inst.cluster_values)
    lay = layouts_from_sizes({3: [5, 7], 11: [12], 40: [5, 7]})
    sched = multiring.build_ring_schedule(lay)
    rng = np.random.Generator(np.random.Philox(key=4))
    add("sparse_cids", sched, {c: rng.normal(0, 1, 12) for c in (40, 3, 11)})

    # --- edge cases -----------------------------------------------------------
    # ring shorter than C: zero-length chunks (test_multiring.py:95-97)
    lay = layouts_from_sizes({c: [2, 1, 9] for c in range(5)})
    sched = multiring.build_ring_schedule(lay)
    rng = np.random.Generator(np.random.Philox(key=6))
    add("short_rings_c5", sched, {c: rng.normal(0, 3, 12) for c in range(5)})
    # special values: signed zeros, subnormals, huge, inf
    lay = layouts_from_sizes({c: [16, 16] for c in range(3)})
    sched = multiring.build_ring_schedule(lay)
    specials = np.array([0.0, -0.0, 5e-324, -5e-324, 1e-310, 1e308, -1e308, np.inf,
                         1.0, -1.0, 3.0, 1e-45, 1.4e-45, -2.5e-40, 7.0, 1e38], dtype=np.float64)
    vals = {
        0: np.concatenate([specials, -specials]),
        1: np.concatenate([specials[::-1], specials]),
        2: np.concatenate([-specials, specials[::-1] * 0.5]),
    }
    add("specials_c3", sched, vals)
    vals = {c: np.full(32, -0.0) for c in range(4)}
    lay = layouts_from_sizes({c: [32] for c in range(4)})
    add("all_neg_zero_c4", multiring.build_ring_schedule(lay), vals)

    np.savez_compressed(os.path.join(HERE, "ring_instances.npz"),
                        names=np.array(names), **store)

    # --- schedule / cost KATs ----------------------------------------------------
    kats = {"schedules": [], "chunk_bounds": [], "cost": []}
    cases = [
        {0: [10, 6], 1: [10, 6]},
        {0: [8, 8], 1: [16]},
        {0: [4, 4, 4], 1: [8, 4], 2: [12]},
        {0: [10], 1: [12]},
        {0: [4, 8], 1: [8, 4]},
        {5: [3, 3, 3, 3], 2: [6, 6], 9: [3, 9]},
        {0: [0, 4], 1: [4]},
    ]
    rng = np.random.Generator(np.random.Philox(key=1234))
    for _ in range(40):
        inst = multiring.random_instance(rng, int(rng.integers(1, 9)), max_peers=5, max_dim=500)
        cases.append({cid: [p.param_len for p in lay] for cid, lay in inst.layouts.items()})
    for sizes in cases:
        lay = layouts_from_sizes(sizes)
        entry = {"sizes": {str(k): v for k, v in sizes.items()}}
        try:
            s = multiring.build_ring_schedule(lay)
            multiring.validate_schedule(s, lay)
            entry["dump"] = s.dump()
            entry["total"] = s.total_params
        except RavnestError as e:
            entry["error"] = type(e).__name__
            entry["message"] = str(e)
        kats["schedules"].append(entry)
    for args in ((0, 10, 3), (5, 2, 4), (0, 0, 3), (7, 100, 7), (3, 17, 8), (0, 25557032, 8)):
        kats["chunk_bounds"].append({"args": list(args), "bounds": multiring.chunk_bounds(*args)})
    for sizes, bw, lat in (({c: [30] for c in range(3)}, 1e6, 0.0),
                           ({c: [512, 512] for c in range(3)}, 1e6, 0.0),
                           ({c: [100, 300] for c in range(2)}, 1e6, 1e-3),
                           ({c: [128] * 5 for c in range(3)}, 1e7, 0.0)):
        s = multiring.build_ring_schedule(layouts_from_sizes(sizes))
        rep = multiring.allreduce_cost(s, bandwidth=bw, latency=lat)
        kats["cost"].append({
            "sizes": {str(k): v for k, v in sizes.items()}, "bandwidth": bw, "latency": lat,
            "rings": [[rc.ring_id, rc.rounds, rc.seg_bytes, rc.bytes_per_member, rc.seconds]
                      for rc in rep.rings],
            "critical": rep.critical_seconds, "single": rep.single_ring_seconds,
        })
    with open(os.path.join(HERE, "schedule_kats.json"), "w") as f:
        json.dump(kats, f, indent=1, sort_keys=True)
    print(f"wrote {len(names)} ring instances, {len(kats['schedules'])} schedule cases")
    make_formats()


def make_formats():
    """Config 1 (BASELINE.json configs[0]): the reference's own session plan
    for the MLP [3072,256,128,10] over two 3-peer clusters, serialised by
    configio.serialize_plan; digests of apply_ring_mean on seeded inputs;
    wire-frame and checkpoint golden bytes (multiring.py:400-426,
    configio.py:495-512)."""
    import hashlib
    import tempfile

    from ravnest import configio, modelcore
    from ravnest.clusterform import ModelFootprint, plan_session
    from ravnest.simnet import NodeSpec

    arch = [3072, 256, 128, 10]
    model, _ = modelcore.build_model(arch, 3, "tanh", "mse")
    fp = ModelFootprint.from_model(model, 2)
    pool, assignment = [], []
    for ci, count in enumerate([3, 3], start=1):
        for j in range(count):
            pool.append(NodeSpec(f"c{ci}n{j}", fp.M, 1e9, 1.0))
            assignment.append(ci)
    plan = plan_session(pool, fp, 2, model, assignment=assignment)
    text = configio.serialize_plan(plan)
    with open(os.path.join(HERE, "config1_plan.txt"), "w") as f:
        f.write(text)
    out = {"ring_lengths": [r.length for r in plan.ring_schedule.rings], "total": plan.ring_schedule.total_params,
           "cases": []}
    for key in (1, 2):
        rng = np.random.Generator(np.random.Philox(key=key))
        vals = {cid: rng.normal(0.0, 1.0, plan.ring_schedule.total_params) for cid in plan.cluster_ids}
        res = multiring.apply_ring_mean(plan.ring_schedule, vals)
        out["cases"].append({
            "philox_key": key, "clusters": plan.cluster_ids, "sigma": 1.0,
            "sha256": {str(c): hashlib.sha256(res[c].astype("<f8").tobytes()).hexdigest() for c in res},
            "first": {str(c): [float(v) for v in res[c][:4]] for c in res},
        })
    frames = []
    for kind, rid, rnd, off, payload in (("ring_chunk", 1, 2, 3, [1.0]), ("ring_chunk", 7, 3, 160, [1.5, -2.25, 3.875]),
                                         ("control", 0, 0, 0, [0.0, 0.0]), ("gradient", 4294967295, 5, 2**40, [-0.0, 5e-324])):
        b = multiring.encode_frame(kind, rid, rnd, off, np.array(payload))
        frames.append({"kind": kind, "ring_id": rid, "round": rnd, "offset": off, "payload": payload, "hex": b.hex()})
    out["frames"] = frames
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "x.ckpt")
        configio.write_checkpoint(path, np.array([1.0, -2.5, 3e-300]))
        with open(path, "rb") as f:
            out["checkpoint_hex"] = f.read().hex()
    with open(os.path.join(HERE, "formats.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote config1_plan.txt, formats.json", out["ring_lengths"])


if __name__ == "__main__":
    main()
