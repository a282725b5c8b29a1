import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# the loopback tests drive several ranks' kernels concurrently on one GPU:
# give every stream its own hardware queue (must be set before CUDA starts)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
REFERENCE_SRC = "/root/reference/pkg/src"  # dev container only; absent on GPU boxes
REFERENCE_INSTALL = os.path.join(ROOT, "baseline", "_ref")  # offline install; travels to the GPU box


def reference_path():
    """Where the unmodified reference can be imported from: the offline
    install in baseline/_ref (dev container and GPU box), else the read-only
    tree of the dev container; None when neither exists."""
    for path in (REFERENCE_INSTALL, REFERENCE_SRC):
        if os.path.isdir(os.path.join(path, "ravnest")):
            return path
    return None


def import_reference(module: str = "ravnest"):
    """The unmodified reference package (CPU checks, the seam tests), or skip."""
    path = reference_path()
    if path is None:
        pytest.skip("reference not present here (baseline/_ref not installed)")
    sys.dont_write_bytecode = True
    if path not in sys.path:
        sys.path.append(path)
    import importlib

    return importlib.import_module(module)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def bits_equal(a, b) -> bool:
    """Bitwise equality of float arrays; any NaN matches any NaN (GPU NaNs are
    canonical, numpy propagates payloads)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.size == 0:
        return True
    ut = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    nan = np.isnan(a)
    if not np.array_equal(nan, np.isnan(b)):
        return False
    return bool(np.array_equal(a.view(ut)[~nan], b.view(ut)[~nan]))


class GoldenInstance:
    def __init__(self, z, name):
        self.name = name
        self.starts = z[f"{name}/starts"]
        self.lens = z[f"{name}/lens"]
        self.cids = z[f"{name}/cids"]
        self.x = z[f"{name}/x"]
        self.apply_ring_mean = z[f"{name}/apply_ring_mean"]
        self.run_allreduce = z[f"{name}/run_allreduce"] if f"{name}/run_allreduce" in z else None
        self.rounds = z[f"{name}/rounds"] if f"{name}/rounds" in z else None
        self.messages = z[f"{name}/messages"] if f"{name}/messages" in z else None
        self.x32 = z[f"{name}/x32"]
        self.apply_ring_mean_f32in = z[f"{name}/apply_ring_mean_f32in"]

    @property
    def c(self):
        return len(self.cids)

    @property
    def total(self):
        return int(self.lens.sum())


def load_instances():
    with np.load(os.path.join(GOLDEN, "ring_instances.npz")) as z:
        names = [str(n) for n in z["names"]]
        data = {k: z[k] for k in z.files}
    return [GoldenInstance(data, n) for n in names]


def load_schedule_kats():
    with open(os.path.join(GOLDEN, "schedule_kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_instances():
    return load_instances()


@pytest.fixture(scope="session")
def schedule_kats():
    return load_schedule_kats()
