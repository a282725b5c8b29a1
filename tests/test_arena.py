"""Zero-copy arena and the tensor-boundary ring split (CPU)."""

import pytest
import torch

from paper_2401_01728_b200 import arena
from bench import WORKLOADS


def _sizes(build):
    with torch.device("meta"):
        m = build()
    return [p.numel() for p in m.parameters()]


def test_ring_split_reproduces_workload_tables():
    # SURVEY.md §8a ring lengths: the model zoo's real parameter tensors
    torchvision = pytest.importorskip("torchvision")
    transformers = pytest.importorskip("transformers")
    cases = {
        "resnet50": (lambda: torchvision.models.resnet50(), 4),
        "bert": (lambda: transformers.BertModel(transformers.BertConfig()), 4),
        "gpt2": (lambda: transformers.GPT2LMHeadModel(transformers.GPT2Config(n_embd=1024, n_layer=24, n_head=16)), 8),
    }
    for name, (build, r) in cases.items():
        sizes = _sizes(build)
        assert arena.tensor_boundary_rings(sizes, r) == WORKLOADS[name], name


def test_arena_views_are_zero_copy():
    torch.manual_seed(0)
    m = torch.nn.Sequential(torch.nn.Linear(7, 5), torch.nn.Tanh(), torch.nn.Linear(5, 3))
    x = torch.randn(4, 7)
    y0 = m(x)
    a = arena.ParamArena(m, grads=True)
    assert a.numel == 7 * 5 + 5 + 5 * 3 + 3
    assert torch.equal(m(x), y0)                      # same function after flattening
    a.flat.mul_(0.0)                                  # writes through the views
    assert all(float(p.abs().sum()) == 0.0 for p in m.parameters())
    m(x).sum().backward()                             # grads land in the flat grad buffer
    assert float(a.grad.abs().sum()) > 0
    sched = a.schedule([3, 1], 2)
    assert [r.length for r in sched.rings] == a.ring_lengths(2)
    assert sched.rings[0].members == ((1, 0), (3, 0))
    assert sched.total_params == a.numel


def test_split_edge_cases():
    assert arena.tensor_boundary_rings([10], 3) == [10]
    assert arena.tensor_boundary_rings([1, 1, 1, 1], 2) == [2, 2]
    assert arena.tensor_boundary_rings([100, 1, 1], 2) == [100, 2]
    with pytest.raises(ValueError):
        arena.tensor_boundary_rings([1], 0)
