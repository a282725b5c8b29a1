"""The push kernel's work order (rv_kernels.cuh, ring_push_kernel), restated:
every item appears exactly once and waits only on items at earlier
positions, which is what lets a co-resident grid taking items in position
order always drain (push transport).  CPU only."""

import random

import pytest


def work_order(C, ua, blag, fused):
    """Position -> item, as the kernel maps it: ('s', unit, peer) scatter,
    ('f', unit) fold, ('b', unit, peer) blend of another owner's unit."""
    head = ua * (C - 1)
    n = head + (ua + blag) * C if fused else ua * C
    out = []
    for w in range(n):
        if w < head:
            out.append(("s", w // (C - 1), w % (C - 1)))
        elif not fused:
            out.append(("f", w - head))
        elif (w - head) % C == 0:
            out.append(("f", (w - head) // C))
        else:
            u = (w - head) // C - blag
            out.append(("b", u, (w - head) % C - 1) if 0 <= u < ua else None)
    return out


@pytest.mark.parametrize("fused", [False, True])
def test_every_item_once_and_dependencies_earlier(fused):
    rng = random.Random(7)
    for _ in range(400):
        C, ua, blag = rng.randint(2, 16), rng.randint(1, 30), rng.randint(0, 40)
        order = work_order(C, ua, blag, fused)
        pos = {}
        for w, item in enumerate(order):
            if item is None or (item[0] == "f" and item[1] >= ua):
                continue  # skipped slots
            assert item not in pos
            pos[item] = w
        scatters = [k for k in pos if k[0] == "s"]
        folds = [k for k in pos if k[0] == "f"]
        blends = [k for k in pos if k[0] == "b"]
        assert len(scatters) == ua * (C - 1) and len(folds) == ua
        assert len(blends) == (ua * (C - 1) if fused else 0)
        for u in range(ua):
            # a fold waits for every peer's scatter of its unit
            assert all(pos[("s", u, r)] < pos[("f", u)] for r in range(C - 1))
            # a blend waits for the owner's fold of its unit (same position
            # map on every rank)
            for r in range(C - 1 if fused else 0):
                assert pos[("f", u)] < pos[("b", u, r)]


def test_split_blend_equals_one_pass_blend():
    """The push kernel's fused blend of another owner's chunk runs in two
    halves -- live <- delta(live, snap) in the scatter item, live <- mean +
    live once the owner's means land -- where delta stores -0.0 for
    bitwise-equal live and snap.  That is bit for bit the one-pass blend
    mean + (live - snap), exactly mean where live == snap (oracle.blend),
    signed zeros, infinities and NaN included."""
    import numpy as np

    from oracle import ring_oracle

    rng = np.random.Generator(np.random.Philox(key=12))
    for dt in (np.float32, np.float64):
        n = 1 << 16
        snap = rng.normal(0, 1, n).astype(dt)
        live = snap + rng.normal(0, 1e-3, n).astype(dt)
        mean = rng.normal(0, 1, n).astype(dt)
        live[::5] = snap[::5]
        special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 1.0], dtype=dt)
        k = len(special)
        grid = np.array(np.meshgrid(np.arange(k), np.arange(k), np.arange(k))).reshape(3, -1)
        mean = np.concatenate([mean, special[grid[0]]])
        live = np.concatenate([live, special[grid[1]]])
        snap = np.concatenate([snap, special[grid[2]]])
        ut = {4: np.uint32, 8: np.uint64}[np.dtype(dt).itemsize]
        with np.errstate(all="ignore"):
            delta = np.where(live.view(ut) == snap.view(ut), dt(-0.0), live - snap)
            two_half = mean + delta
            want = ring_oracle.blend(mean, live, snap)
        nan = np.isnan(want)
        assert np.array_equal(np.isnan(two_half), nan)
        assert np.array_equal(two_half.view(ut)[~nan], want.view(ut)[~nan]), dt
