"""CPU oracle for the multi-ring parameter average -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The shipped path
(``paper_2401_01728_b200``) never imports anything under ``oracle/`` and
fails loudly when its CUDA library is missing.

What it restates (reference = /root/reference/pkg/src/ravnest):

* ``chunk_bounds`` -- ``multiring.py:134-144``: a ring of ``length`` params is
  cut into C contiguous chunks, ``base, rem = divmod(length, C)``, chunk i
  gets ``base + (i < rem)`` elements.
* ``ring_mean`` -- the arithmetic of ``apply_ring_mean`` (``multiring.py:302-333``)
  and of ``AllReduceController.handle`` (``multiring.py:216-221``), written in
  closed form.  In reduce-scatter round r member m sends chunk (m - r) mod C to
  member m+1, which does ``seg += payload``; so chunk k is accumulated by the
  members k, k+1, ..., k+C-1 (mod C) in that order, and the member that
  receives it in round C-2 divides by C (``multiring.py:218-219``).  The
  all-gather rounds then copy those bits to every member (``:220-221``).
  Hence, for every member::

      out[k-chunk] = fl( fl(...fl(x_k + x_{k+1}) ... + x_{k+C-1}) / C )

  with x_m the vector of the m-th smallest cluster id.  Every add is the
  IEEE add of the working dtype; the divide is IEEE true division.
* ``ring_mean_rounds`` -- an independent round-by-round simulation of the
  same ring (message order of ``apply_ring_mean``), dtype-generic; used by
  the tests to cross-check the closed form, and to derive the fp32
  ring-order oracle (the reference itself always works in float64,
  ``multiring.py:309``).
* ``mean_reference`` -- ``oracle.py:152-161`` (scalar loop in input order,
  the reference's own tolerance oracle).

Parity pinning: ``tests/golden/*.npz`` are produced by
``tests/golden/make_golden.py`` from the unmodified reference
(``apply_ring_mean`` / ``run_allreduce``); ``tests/test_oracle.py`` asserts
this module and the C restatement (``ring_oracle.c``) are bitwise equal to
them.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

ACC_F64 = "f64"        # reference-exact: fold in float64 (multiring.py:309 casts to float64)
ACC_NATIVE = "native"  # fold in the storage dtype (fp32 ring order)


def chunk_bounds(start: int, length: int, c: int) -> list[tuple[int, int]]:
    """Chunk boundaries of one ring (restates multiring.py:134-144)."""
    base, rem = divmod(int(length), int(c))
    out = []
    lo = int(start)
    for i in range(int(c)):
        n = base + (1 if i < rem else 0)
        out.append((lo, lo + n))
        lo += n
    return out


def ring_mean(
    ring_starts: Sequence[int],
    ring_lens: Sequence[int],
    values: Sequence[np.ndarray],
    acc: str = ACC_F64,
) -> list[np.ndarray]:
    """Closed-form multi-ring mean.

    ``values[m]`` is the flat vector of the m-th smallest cluster id.  With
    ``acc == "f64"`` the inputs are widened to float64 and the result is
    float64 -- exactly ``apply_ring_mean`` (multiring.py:302-333).  With
    ``acc == "native"`` the fold runs in the input dtype (fp32 ring order).
    """
    c = len(values)
    if acc == ACC_F64:
        work = [np.asarray(v, dtype=np.float64) for v in values]
        dt = np.float64
    elif acc == ACC_NATIVE:
        dt = np.asarray(values[0]).dtype.type
        work = [np.asarray(v, dtype=dt) for v in values]
    else:
        raise ValueError(f"unknown accumulation mode {acc!r}")
    out = [w.copy() for w in work]
    if c < 2:
        return out
    divisor = dt(c)
    for start, length in zip(ring_starts, ring_lens):
        for k, (lo, hi) in enumerate(chunk_bounds(start, length, c)):
            if hi == lo:
                continue
            s = work[k][lo:hi].copy()
            for j in range(1, c):
                s = s + work[(k + j) % c][lo:hi]
            s = s / divisor
            for m in range(c):
                out[m][lo:hi] = s
    return out


def ring_mean_rounds(
    ring_starts: Sequence[int],
    ring_lens: Sequence[int],
    values: Sequence[np.ndarray],
    dtype=np.float64,
) -> list[np.ndarray]:
    """Round-by-round ring (message order of multiring.py:310-332), any dtype.

    Each round every member posts one chunk to its successor; all posts of a
    round are taken before any is applied.  Reduce-scatter rounds add (and
    the last one divides by C); all-gather rounds overwrite.
    """
    c = len(values)
    work = [np.array(v, dtype=dtype) for v in values]
    if c < 2:
        return work
    for start, length in zip(ring_starts, ring_lens):
        bounds = chunk_bounds(start, length, c)
        for rnd in range(2 * (c - 1)):
            reduce_phase = rnd < c - 1
            posts = []
            for m in range(c):
                k = (m - rnd) % c if reduce_phase else (m + 1 - (rnd - (c - 1))) % c
                lo, hi = bounds[k]
                posts.append((k, work[m][lo:hi].copy()))
            for m, (k, payload) in enumerate(posts):
                lo, hi = bounds[k]
                seg = work[(m + 1) % c][lo:hi]  # view: the updates land in place
                if reduce_phase:
                    seg += payload
                    if rnd == c - 2:
                        seg /= dtype(c)
                else:
                    seg[...] = payload
    return work


def mean_reference(vectors: Sequence[np.ndarray]) -> np.ndarray:
    """Scalar-loop mean in input order (restates oracle.py:152-161)."""
    n = len(vectors[0])
    out = np.empty(n, dtype=np.float64)
    inv = float(len(vectors))
    for i in range(n):
        s = 0.0
        for v in vectors:
            s += float(v[i])
        out[i] = s / inv
    return out


def blend(mean: np.ndarray, live: np.ndarray, snap: np.ndarray) -> np.ndarray:
    """Delayed-update blend ``live <- mean + (live - snap)``.

    In-flight updates computed on the stale snapshot land on the averaged
    parameters, as ``pipeline.py:384-411`` applies stale gradients to the
    post-average live values.  Where ``live`` equals ``snap`` bit for bit the
    result is ``mean`` itself (keeps -0.0, as the reference's zero-time
    snapshot would).  Two roundings, in the storage dtype.
    """
    live = np.asarray(live)
    snap = np.asarray(snap)
    mean = np.asarray(mean, dtype=live.dtype)
    utype = {4: np.uint32, 8: np.uint64}[live.dtype.itemsize]
    same = live.view(utype) == snap.view(utype)
    d = live - snap
    out = mean + d
    out[same] = mean[same]
    return out


def floor1_rel_err(got: np.ndarray, want: np.ndarray) -> float:
    """The reference's tolerance metric |got-want| / max(|want|, 1)
    (test_multiring.py:125, test_acceptance.py:41, oracle.py:374)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.size == 0:
        return 0.0
    return float((np.abs(got - want) / np.maximum(np.abs(want), 1.0)).max())


def random_instance(rng: np.random.Generator, n_clusters: int, max_peers: int = 4, max_dim: int = 4096):
    """Restates multiring.random_instance (multiring.py:440-465): random nested
    per-cluster layouts and N(0, 10) cluster vectors, drawing from ``rng`` in
    the same order, so a Philox key reproduces the reference's instance
    stream (pinned against tests/golden crit1_* fixtures).  Returns
    (layouts {cid: [(start, len), ...]}, values {cid: float64[dim]})."""
    p_max = int(rng.integers(1, max_peers + 1))
    lo = max(p_max, 2)
    dim = max(int(np.exp(rng.uniform(np.log(lo), np.log(max_dim)))), p_max)
    master = sorted(rng.choice(np.arange(1, dim), size=p_max - 1, replace=False).tolist()) if p_max > 1 else []
    layouts = {}
    for cid in range(n_clusters):
        cuts = list(master) if cid == 0 else [c for c in master if rng.random() < 0.5]
        edges = [0, *cuts, dim]
        layouts[cid] = [(edges[i], edges[i + 1] - edges[i]) for i in range(len(edges) - 1)]
    values = {cid: rng.normal(0.0, 10.0, size=dim) for cid in range(n_clusters)}
    return layouts, values


def rings_of_layouts(layouts) -> tuple[list[int], list[int]]:
    """Ring (start, length) lists for nested layouts: the union of all
    clusters' cuts (multiring.py:80-105)."""
    cuts = sorted({s for lay in layouts.values() for s, _ in lay if s > 0})
    total = sum(n for _, n in next(iter(layouts.values())))
    edges = [0, *cuts, total]
    return edges[:-1], [edges[i + 1] - edges[i] for i in range(len(edges) - 1)]
