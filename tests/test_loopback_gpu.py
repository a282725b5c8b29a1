"""The multi-rank transports (pull, push, LL, push with the fused blend) on ONE
GPU: C rank plans on cuda:0 (paper_2401_01728_b200.loopback), each rank on
its own streams with 1/C of the SMs.  These are the kernels, flags and work
orders every rank of an N-GPU job runs (DistRingGroup); here they are
checked bit for bit against the reference-generated fixtures and the oracle
on a one-GPU box.

Bars, per transport:
  * float64                 == unmodified reference apply_ring_mean, bitwise
  * float32, f64 fold       == float32(reference on the fp32 inputs), bitwise
  * float32, native fold    == fp32 ring-order closed form, bitwise
  * fused blend             == oracle blend(mean, live, snap), bitwise
Reference: multiring.py:302-333 (arithmetic), :185-225 (the ring exchange
these transports replace), pipeline.py:384-411 (the delayed-update blend).
"""

import numpy as np
import pytest

from conftest import bits_equal, host_threads
from oracle import c_oracle, ring_oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2401_01728_b200.errors import StallError  # noqa: E402
from paper_2401_01728_b200.loopback import LoopbackGroup  # noqa: E402

SENTINEL = -1234.5
GUARD = 8
TIMEOUT_S = 10.0  # a transport that cannot make progress fails the test instead of hanging the box


def starts_of(lens):
    return [int(s) for s in np.cumsum([0] + list(lens[:-1]))]


class Members:
    """C member buffers with sentinel guard bands (compute-sanitizer is
    closed on this pool: an out-of-bounds write shows in the bands)."""

    def __init__(self, rows, dtype, offsets=None):
        self.total = len(rows[0])
        self.bufs, self.offs, self.views = [], [], []
        for m, r in enumerate(rows):
            off = GUARD + (0 if offsets is None else offsets[m])
            buf = torch.full((self.total + off + GUARD,), SENTINEL, dtype=dtype, device="cuda:0")
            v = buf[off:off + self.total]
            v.copy_(torch.from_numpy(np.ascontiguousarray(r)))
            self.bufs.append(buf)
            self.offs.append(off)
            self.views.append(v)

    def fill(self, rows):
        for v, r in zip(self.views, rows):
            v.copy_(torch.from_numpy(np.ascontiguousarray(r)))

    def guards_ok(self):
        for buf, off in zip(self.bufs, self.offs):
            h = buf.cpu().numpy()
            if not ((h[:off] == SENTINEL).all() and (h[off + self.total:] == SENTINEL).all()):
                return False
        return True

    def host(self):
        return np.stack([v.cpu().numpy() for v in self.views])


def loopback_mean(proto, starts, lens, rows, dtype, acc="f64", lanes=1, offsets=None, src_ne_dst=False,
                  options=None):
    """One cycle through a LoopbackGroup; returns (means as host rows, guards ok)."""
    src = Members(rows, dtype, offsets)
    dst = Members([np.full(len(rows[0]), np.nan, dtype=rows[0].dtype)] * len(rows), dtype, offsets) \
        if src_ne_dst else None
    g = LoopbackGroup(starts, lens, sum(lens), len(rows), dtype, protocol=proto, acc=acc, lanes=lanes,
                      options=options, timeout_s=TIMEOUT_S)
    try:
        g.bind_tensors(src.views, None if dst is None else dst.views)
        g.run()
        torch.cuda.synchronize()
        g.check()
    finally:
        g.close()
    out = (dst or src)
    return out.host(), src.guards_ok() and (dst is None or dst.guards_ok())


# ---------------------------------------------------------------------------
# reference-generated fixtures (tests/golden, make_golden.py)


@pytest.mark.parametrize("proto", ["pull", "push", "ll"])
def test_golden_fixtures_every_transport(golden_instances, proto):
    for g in golden_instances:
        if g.c < 2 or g.total == 0:
            continue
        starts, lens = [int(s) for s in g.starts], [int(n) for n in g.lens]
        if proto != "ll":  # LL carries fp32 only
            got, ok = loopback_mean(proto, starts, lens, list(g.x), torch.float64)
            assert ok and bits_equal(got, g.apply_ring_mean), (g.name, "f64")
        got, ok = loopback_mean(proto, starts, lens, list(g.x32), torch.float32)
        with np.errstate(over="ignore"):
            want = g.apply_ring_mean_f32in.astype(np.float32)
        assert ok and bits_equal(got, want), (g.name, "f32/f64 fold")
        got, ok = loopback_mean(proto, starts, lens, list(g.x32), torch.float32, acc="native")
        want = np.stack(ring_oracle.ring_mean(g.starts, g.lens, list(g.x32), acc="native"))
        assert ok and bits_equal(got, want), (g.name, "f32 native")


# ---------------------------------------------------------------------------
# seeded layouts: ragged / zero-length rings, lanes, alignment classes, src != dst


def random_layouts(c):
    rng = np.random.Generator(np.random.Philox(key=77 + c))
    out = []
    for _ in range(3):
        n_rings = int(rng.integers(1, 9))
        lens = [int(x) for x in rng.integers(0, 200000, n_rings)]
        lens[0] += c - 1
        out.append(lens)
    out.append([1, 0, 2, c + 1, 3 * c - 1])  # tiny and zero-length rings
    return out


@pytest.mark.parametrize("c", [2, 3, 4, 8])
@pytest.mark.parametrize("proto", ["pull", "push", "ll"])
def test_transports_random_layouts(proto, c):
    for li, lens in enumerate(random_layouts(c)):
        starts, total = starts_of(lens), sum(lens)
        variants = [("f64", torch.float32, 1, None, False), ("native", torch.float32, 1, None, False),
                    ("f64", torch.float32, len(lens), None, True), ("f64", torch.float32, 2 * len(lens) + 1, None, False),
                    ("f64", torch.float32, 1, [1] * c, False), ("f64", torch.float32, 1, [m % 3 for m in range(c)], False)]
        if proto != "ll":
            variants += [("f64", torch.float64, 1, None, False), ("f64", torch.float64, 3, [1] * c, True)]
        for acc, dt, lanes, offsets, src_ne_dst in variants:
            npdt = np.float32 if dt == torch.float32 else np.float64
            rows = [np.random.Generator(np.random.Philox(key=1000 * li + m)).normal(0, 1, total).astype(npdt)
                    for m in range(c)]
            want = np.stack(ring_oracle.ring_mean(starts, lens, rows, acc=acc)).astype(npdt)
            got, ok = loopback_mean(proto, starts, lens, rows, dt, acc=acc, lanes=lanes, offsets=offsets,
                                    src_ne_dst=src_ne_dst)
            tag = (proto, c, li, acc, str(dt), lanes, offsets, src_ne_dst)
            assert ok, ("write outside the member vector",) + tag
            assert bits_equal(got, want), tag


@pytest.mark.parametrize("proto", ["pull", "push", "ll"])
def test_back_to_back_cycles_and_graph_replay(proto):
    """Three cycles with no host sync in between, then a captured cycle
    replayed twice: device-side epochs, work counters and flags advance
    consistently (graph-safe)."""
    c, lens = 4, [200003, 5, 77777, 9]
    starts, total = starts_of(lens), sum(lens)
    rows = [np.random.Generator(np.random.Philox(key=900 + m)).normal(0, 1, total).astype(np.float32)
            for m in range(c)]
    mem = Members(rows, torch.float32)
    g = LoopbackGroup(starts, lens, total, c, torch.float32, protocol=proto, timeout_s=TIMEOUT_S)
    try:
        g.bind_tensors(mem.views)
        for _ in range(3):
            g.run()
        torch.cuda.synchronize()
        g.check()
        cur = rows
        for _ in range(3):
            cur = [v.astype(np.float32) for v in ring_oracle.ring_mean(starts, lens, cur)]
        assert bits_equal(mem.host(), np.stack(cur))
        mem.fill(rows)
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            g.run(after=cap)
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
        g.check()
        cur = rows
        for _ in range(2):
            cur = [v.astype(np.float32) for v in ring_oracle.ring_mean(starts, lens, cur)]
        assert bits_equal(mem.host(), np.stack(cur)) and mem.guards_ok()
    finally:
        g.close()


# ---------------------------------------------------------------------------
# delayed-update blend inside the cycle (push: fused per unit; pull / LL: per lane)


@pytest.mark.parametrize("c", [2, 3, 8])
@pytest.mark.parametrize("proto", ["push", "pull", "ll"])
def test_fused_blend(proto, c):
    lens = [200003, 5, 77777, 2 * c + 1]
    starts, total = starts_of(lens), sum(lens)
    for dt, lanes in ((torch.float32, 1), (torch.float32, 3), (torch.float64, 1)):
        if proto == "ll" and dt == torch.float64:
            continue
        npdt = np.float32 if dt == torch.float32 else np.float64
        snaps = [np.random.Generator(np.random.Philox(key=500 + m)).normal(0, 1, total).astype(npdt)
                 for m in range(c)]
        lives = [s + np.random.Generator(np.random.Philox(key=600 + m)).normal(0, 1e-3, total).astype(npdt)
                 for m, s in enumerate(snaps)]
        for m in range(c):  # entries untouched since the snapshot: exactly the mean there
            lives[m][::7] = snaps[m][::7]
        src = Members(snaps, dt)
        mean = Members([np.full(total, np.nan, dtype=npdt)] * c, dt)
        live = Members(lives, dt)
        g = LoopbackGroup(starts, lens, total, c, dt, protocol=proto, lanes=lanes, timeout_s=TIMEOUT_S)
        try:
            g.bind_tensors(src.views, mean.views)
            g.bind_live(live.views)
            for _ in range(3):
                g.run()
            torch.cuda.synchronize()
            g.check()
        finally:
            g.close()
        want_mean = np.stack(ring_oracle.ring_mean(starts, lens, snaps)).astype(npdt)
        want_live = [lv for lv in lives]
        for _ in range(3):
            want_live = [ring_oracle.blend(want_mean[m], want_live[m], snaps[m]) for m in range(c)]
        tag = (proto, c, str(dt), lanes)
        assert bits_equal(mean.host(), want_mean), tag
        assert bits_equal(live.host(), np.stack(want_live)), tag
        assert bits_equal(src.host(), np.stack(snaps)), ("snapshot modified",) + tag
        assert src.guards_ok() and mean.guards_ok() and live.guards_ok(), tag


# ---------------------------------------------------------------------------
# the kernel buckets of 8- and 16-GPU jobs (RV_OPT_MIN_CB), odd member counts


@pytest.mark.parametrize("min_cb", [8, 16])
@pytest.mark.parametrize("proto", ["pull", "push", "ll"])
def test_wider_kernel_buckets(proto, min_cb):
    for c in (2, 3, 5):
        lens = [100003, 7, 4096 + 5, 3 * c + 1]
        starts, total = starts_of(lens), sum(lens)
        rows = [np.random.Generator(np.random.Philox(key=300 + m)).normal(0, 3, total).astype(np.float32)
                for m in range(c)]
        for acc in ("f64", "native"):
            want = np.stack(ring_oracle.ring_mean(starts, lens, rows, acc=acc)).astype(np.float32)
            got, ok = loopback_mean(proto, starts, lens, rows, torch.float32, acc=acc, options={"min_cb": min_cb})
            assert ok and bits_equal(got, want), (proto, min_cb, c, acc)


# ---------------------------------------------------------------------------
# the north-star transport at size: BERT-base rings, C = 8 ranks, push


def test_bert_c8_push_every_element():
    """BERT-base tensor-boundary rings, 8 ranks on the push
    transport (the CB = 8 kernel an 8-GPU job runs), every element against the
    C oracle (f32 in, f64 fold, f32 out)."""
    lens = [26201088, 27168768, 27170304, 28942080]
    c, starts, total = 8, starts_of(lens), sum(lens)
    gen = torch.Generator(device="cuda").manual_seed(8)
    xs = [torch.randn(total, device="cuda", generator=gen) * 0.02 for _ in range(c)]
    rows = [x.cpu().numpy() for x in xs]
    want = np.empty_like(rows[0])  # every member ends with the same bits: one output, written C times
    c_oracle.ring_mean_into(c_oracle.MODE_F32_ACC64, starts, lens, rows, None, [want] * c, threads=host_threads())
    g = LoopbackGroup(starts, lens, total, c, torch.float32, protocol="push", timeout_s=TIMEOUT_S)
    try:
        g.bind_tensors(xs)
        g.run()
        torch.cuda.synchronize()
        g.check()
    finally:
        g.close()
    for m in range(c):
        assert np.array_equal(xs[m].cpu().numpy().view(np.uint32), want.view(np.uint32)), m


# ---------------------------------------------------------------------------
# failure detection


@pytest.mark.parametrize("proto", ["pull", "push", "ll"])
def test_missing_rank_times_out_and_reports(proto):
    """Only rank 0 launches: its kernel gives up after the timeout with a
    StallError naming a missing rank (no hang), the non-blocking failure word
    is up, and after a reset the full group averages correctly."""
    c, lens = 3, [4097, 333]
    starts, total = starts_of(lens), sum(lens)
    rows = [np.full(total, float(m), dtype=np.float32) for m in range(c)]
    mem = Members(rows, torch.float32)
    g = LoopbackGroup(starts, lens, total, c, torch.float32, protocol=proto, timeout_s=0.5)
    try:
        g.bind_tensors(mem.views)
        assert not g.failed()
        g.plans[0].run([g.streams[0]])
        torch.cuda.synchronize()
        assert g.plans[0].failed()
        with pytest.raises(StallError, match="rank"):
            g.plans[0].check_status()
    finally:
        g.close()
    # a fresh group works
    mem.fill(rows)
    g = LoopbackGroup(starts, lens, total, c, torch.float32, protocol=proto, timeout_s=TIMEOUT_S)
    try:
        g.bind_tensors(mem.views)
        g.run()
        torch.cuda.synchronize()
        g.check()
        assert not g.failed()
    finally:
        g.close()
    assert (mem.host() == np.float32(sum(range(c)) / c)).all()


@pytest.mark.multigpu
@pytest.mark.parametrize("proto", ["pull", "push", "ll"])
def test_ranks_spread_over_devices(proto):
    """C = 8 rank plans over every visible GPU in one process (two or more
    ranks per GPU): the 8-rank kernels with real NVLink peer traffic and
    sys-scope flags between devices, bit-exact against the oracle."""
    ng = torch.cuda.device_count()
    if ng < 2:
        pytest.skip("needs >= 2 GPUs")
    c = 8
    devices = [m * ng // c for m in range(c)]
    for li, lens in enumerate(random_layouts(c)[:2] + [[1 << 20, 77777, 3]]):
        starts, total = starts_of(lens), sum(lens)
        rows = [np.random.Generator(np.random.Philox(key=4000 * li + m)).normal(0, 1, total).astype(np.float32)
                for m in range(c)]
        want = np.stack(ring_oracle.ring_mean(starts, lens, rows)).astype(np.float32)
        xs = [torch.from_numpy(r).to(f"cuda:{d}") for r, d in zip(rows, devices)]
        g = LoopbackGroup(starts, lens, total, c, torch.float32, protocol=proto, devices=devices, timeout_s=TIMEOUT_S)
        try:
            g.bind_tensors(xs)
            for _ in range(2):  # two cycles: epochs and staging reuse across devices
                g.run()
            for d in set(devices):
                torch.cuda.synchronize(d)
            g.check()
        finally:
            g.close()
        twice = np.stack(ring_oracle.ring_mean(starts, lens, list(want))).astype(np.float32)
        assert bits_equal(np.stack([x.cpu().numpy() for x in xs]), twice), (proto, li)
