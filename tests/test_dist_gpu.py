"""Multi-process (one process per GPU) parity through DistRingGroup: runs
tests/dist_worker.py under torchrun on every visible GPU (>= 2)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def test_dist_ring_group_parity():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    n = torch.cuda.device_count()
    env = dict(os.environ, RAVNEST_B200_TIMEOUT_S="10")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "tests", "dist_worker.py")]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert f"DIST OK world={n}" in out, out[-4000:]


@pytest.mark.parametrize("world,min_cb", [(3, 0), (0, 8), (0, 16)])
def test_dist_wider_kernel_buckets_and_odd_world(world, min_cb):
    """The CB = 8 / 16 kernel instantiations an 8- or 16-GPU job selects,
    run here with the box's GPUs (the min_cb plan option forces the bucket; the
    kernels loop over the runtime member count), and a 3-rank job (odd C:
    true division, uneven chunks, 2 peers per owner)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    n = world or torch.cuda.device_count()
    if n > torch.cuda.device_count():
        pytest.skip(f"needs {n} GPUs")
    env = dict(os.environ, RAVNEST_B200_TIMEOUT_S="10", RAVNEST_DIST_QUICK="1")
    if min_cb:
        env["RAVNEST_TEST_MIN_CB"] = str(min_cb)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29540 + min_cb + world),
           os.path.join(ROOT, "tests", "dist_worker.py")]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert f"DIST OK world={n}" in out, out[-4000:]


def test_async_averager_matches_reference_semantics():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    n = torch.cuda.device_count()
    env = dict(os.environ, RAVNEST_B200_TIMEOUT_S="10")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29534",
           os.path.join(ROOT, "tests", "dist_averager_worker.py")]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert f"AVERAGER OK world={n}" in out, out[-4000:]
