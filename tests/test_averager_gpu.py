"""AsyncAverager's schedule (orchestrator.py:302-363 with staleness tau,
pipeline.py:384-411) on ONE GPU: C clusters trained in lock-step in one
process (LocalAsyncAverager), averaged every kappa updates on a side stream
-- co-resident (TMA kernel) or through the multi-rank transports with one
rank plan per cluster -- and the tau stale updates blended back.  A shadow
replays every update with the oracle mean + oracle blend at the same points;
the live parameters must match it bit for bit.  (The one-process-per-GPU
AsyncAverager runs the same core in tests/dist_averager_worker.py.)"""

import numpy as np
import pytest

from oracle import ring_oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2401_01728_b200.averager import LocalAsyncAverager  # noqa: E402


def grad(m, t, n):
    g = torch.Generator(device="cuda").manual_seed(1000 * m + t)
    return torch.randn(n, device="cuda", generator=g)


def oracle_cycle(starts, lens, snaps, shadow):
    mean = ring_oracle.ring_mean(starts, lens, [s.cpu().numpy() for s in snaps])
    return [torch.from_numpy(ring_oracle.blend(mean[m].astype(np.float32), shadow[m].cpu().numpy(),
                                               snaps[m].cpu().numpy())).cuda() for m in range(len(shadow))]


@pytest.mark.parametrize("kappa,tau,graph,transport", [
    (3, 0, False, "co-resident"), (4, 2, False, "co-resident"), (5, 3, True, "co-resident"),
    (4, 2, False, "push"), (5, 3, True, "push"), (3, 1, False, "pull"), (2, 1, True, "ll"),
])
def test_local_async_averager_matches_reference_semantics(kappa, tau, graph, transport):
    c = 3
    lens = [70001, 3, 33333, 2 * c + 1]
    starts = [int(x) for x in np.cumsum([0] + lens[:-1])]
    n = sum(lens)
    eta = 1e-2
    lives = [torch.randn(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7 + m))
             for m in range(c)]
    shadow = [x.clone() for x in lives]
    avg = LocalAsyncAverager(lives, starts=starts, lens=lens, kappa=kappa, tau=tau, transport=transport, graph=graph)
    snaps, pending = None, None
    steps = 4 * kappa + tau + 1
    for t in range(1, steps + 1):
        avg.before_update()
        with torch.cuda.stream(avg.train_stream):
            for m in range(c):
                lives[m].sub_(grad(m, t, n), alpha=eta)
        avg.step()
        for m in range(c):
            shadow[m].sub_(grad(m, t, n), alpha=eta)
        if pending is not None and t >= pending + tau:
            shadow = oracle_cycle(starts, lens, snaps, shadow)
            pending = None
        if t % kappa == 0 and pending is None:
            snaps = [s.clone() for s in shadow]
            pending = t
            if tau == 0:
                shadow = oracle_cycle(starts, lens, snaps, shadow)
                pending = None
    avg.flush()
    if pending is not None:
        shadow = oracle_cycle(starts, lens, snaps, shadow)
    torch.cuda.synchronize()
    avg.group.check()
    assert not avg.group.failed()
    for m in range(c):
        got = lives[m].cpu().numpy().view(np.uint32)
        want = shadow[m].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want), (m, int((got != want).sum()))
    assert avg.cycles == steps // kappa
    avg.close()
