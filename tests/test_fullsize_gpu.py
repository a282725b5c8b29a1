"""Full-size parity at the BASELINE.json configurations, every element.

SURVEY §8a ring tables (tensor-boundary rings of the named models), C = 8
clusters, fp32 parameters drawn at sigma 0.02 (BERT-style init), 1 and 10
(the stress scales of §8c / random_instance), checked element by element:

  * against the C oracle (f32 in, f64 fold, f32 out): bitwise -- i.e. the
    float32 rounding of the reference's float64 apply_ring_mean;
  * against the float64 reference value on the reference's floor-1 metric
    |got - want| / max(|want|, 1) <= 1e-6 (north_star; test_multiring.py:125)
    on the full vectors.
Config 4 (GPT-2 medium, 8 rings, tau = 4 delayed-update blend) is checked at
full size through the fused co-resident kernel and through the fused push
transport with 8 ranks (LoopbackGroup), against oracle.blend.
"""

import numpy as np
import pytest

from conftest import bits_equal, host_threads
from oracle import c_oracle, ring_oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2401_01728_b200.loopback import LoopbackGroup  # noqa: E402
from paper_2401_01728_b200.plan import LocalRingGroup  # noqa: E402

BERT = [26201088, 27168768, 27170304, 28942080]
GPT2 = [51463168, 43039744, 41987072, 41986048, 41989120, 41987072, 41986048, 50384896]
C = 8
TOL = 1e-6  # north_star: fp32 within 1e-6 of the reference (floor-1 metric)


def starts_of(lens):
    return [int(s) for s in np.cumsum([0] + list(lens[:-1]))]


def device_inputs(total, sigma, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn(total, device="cuda", generator=gen) * sigma for _ in range(C)]


def oracle_means(lens, rows):
    """(float32 result, float64 reference value): one array each -- every
    member ends with the same bits."""
    total = sum(lens)
    out64 = np.empty(total, dtype=np.float64)
    out32 = np.empty(total, dtype=np.float32)
    c_oracle.ring_mean_into(c_oracle.MODE_F32_ACC64, starts_of(lens), lens, rows, [out64] * C, [out32] * C,
                            threads=host_threads())
    return out32, out64


def floor1(got32, want64):
    # chunked: full vectors of up to 355M elements
    worst = 0.0
    for a in range(0, len(want64), 1 << 25):
        worst = max(worst, ring_oracle.floor1_rel_err(got32[a:a + (1 << 25)], want64[a:a + (1 << 25)]))
    return worst


@pytest.mark.parametrize("workload,lens,sigma", [
    ("bert", BERT, 0.02), ("bert", BERT, 1.0), ("bert", BERT, 10.0),
    ("gpt2", GPT2, 0.02), ("gpt2", GPT2, 10.0),
])
def test_co_resident_every_element(workload, lens, sigma):
    total = sum(lens)
    xs = device_inputs(total, sigma, seed=(1000 if workload == "bert" else 2000) + int(sigma * 100))
    rows = [x.cpu().numpy() for x in xs]
    want32, want64 = oracle_means(lens, rows)
    del rows
    g = LocalRingGroup(starts_of(lens), lens, total, [0] * C, torch.float32)
    g.bind_tensors(xs)
    g.run()
    torch.cuda.synchronize()
    g.check()
    g.close()
    for m in range(C):
        got = xs[m].cpu().numpy()
        assert bits_equal(got, want32), (workload, sigma, m)
    err = floor1(got, want64)
    assert err <= TOL, (workload, sigma, err)
    assert err <= 2.0 ** -24  # f64 fold: one rounding, <= half an fp32 ulp relative


def stale_pair(total, seed, tau=4, eta=1e-3):
    """snapshot ~ N(0, 0.02); live = snap - eta * sum of
    tau N(0, 1) updates, with every 7th entry untouched since the snapshot
    (the blend must write exactly the mean there)."""
    gen = torch.Generator(device="cuda").manual_seed(seed)
    snaps, lives = [], []
    for _ in range(C):
        s = torch.randn(total, device="cuda", generator=gen) * 0.02
        live = s.clone()
        for _ in range(tau):
            live.sub_(torch.randn(total, device="cuda", generator=gen), alpha=eta)
        live[::7] = s[::7]
        snaps.append(s)
        lives.append(live)
    return snaps, lives


def check_blend(lens, snaps, lives_before, means, lives_after):
    rows = [s.cpu().numpy() for s in snaps]
    want32, _ = oracle_means(lens, rows)
    for m in range(C):
        assert bits_equal(means[m].cpu().numpy(), want32), ("mean", m)
        want_live = ring_oracle.blend(want32, lives_before[m], rows[m])
        assert bits_equal(lives_after[m].cpu().numpy(), want_live), ("live", m)


def test_config4_gpt2_fused_blend_co_resident():
    total = sum(GPT2)
    snaps, lives = stale_pair(total, seed=4)
    before = [lv.cpu().numpy() for lv in lives]
    means = [torch.empty_like(s) for s in snaps]
    g = LocalRingGroup(starts_of(GPT2), GPT2, total, [0] * C, torch.float32)
    g.bind_tensors(snaps, means)
    g.bind_live(lives)  # fused into the co-resident TMA kernel
    g.run()
    torch.cuda.synchronize()
    g.check()
    g.close()
    check_blend(GPT2, snaps, before, means, lives)


def test_config4_gpt2_fused_blend_push_8_ranks():
    """The kernel config 4 runs on 8 GPUs (push, CB = 8, fused blend), with
    the 8 ranks on one device."""
    total = sum(GPT2)
    snaps, lives = stale_pair(total, seed=5)
    before = [lv.cpu().numpy() for lv in lives]
    means = [torch.empty_like(s) for s in snaps]
    g = LoopbackGroup(starts_of(GPT2), GPT2, total, C, torch.float32, protocol="push", timeout_s=30.0)
    try:
        g.bind_tensors(snaps, means)
        g.bind_live(lives)
        g.run()
        torch.cuda.synchronize()
        g.check()
    finally:
        g.close()
    check_blend(GPT2, snaps, before, means, lives)
