"""CPU-side checks of the C ABI library: it loads without a GPU and exports
every symbol include/ravnest_b200.h declares; status codes map onto the
reference's exception classes."""

import os
import re

import pytest

from conftest import ROOT

import paper_2401_01728_b200 as rv
from paper_2401_01728_b200 import _native


def header_symbols():
    with open(os.path.join(ROOT, "include", "ravnest_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^(?:int|const char \*|size_t)\s*\*?\s*(rv_\w+)\(", text, re.M)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for name in ("rv_plan_create", "rv_plan_bind", "rv_allreduce_mean", "rv_allreduce_mean_host",
                 "rv_plan_destroy", "rv_last_error", "rv_version", "rv_blend", "rv_ipc_export"):
        assert name in syms


def test_library_loads_and_exports_every_header_symbol():
    lib = _native.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, name
    assert lib.rv_version() == 1
    assert lib.rv_ipc_handle_size() == 64


def test_library_is_in_tree():
    assert os.path.dirname(_native.LIB_PATH) == os.path.join(ROOT, "paper_2401_01728_b200")


def test_status_strings():
    lib = _native.load()
    assert lib.rv_status_string(_native.RV_E_TIMEOUT) == b"peer stall (timeout)"


@pytest.mark.parametrize("code,exc", [(_native.RV_E_CONFIG, rv.ConfigError), (_native.RV_E_LAYOUT, rv.LayoutError),
                                      (_native.RV_E_TIMEOUT, rv.StallError), (_native.RV_E_CUDA, rv.RavnestError),
                                      (_native.RV_E_ARG, rv.RavnestError)])
def test_status_mapping(code, exc):
    with pytest.raises(exc):
        _native.check(code, "x")


def test_plan_create_validates_before_touching_cuda():
    # argument errors are reported even where no device exists
    import ctypes

    lib = _native.load()
    h = ctypes.c_void_p()
    rs = (ctypes.c_int64 * 1)(0)
    rl = (ctypes.c_int64 * 1)(10)
    assert lib.rv_plan_create(ctypes.byref(h), 0, 1, 1, rs, rl, 10, 0, 0) == _native.RV_E_CONFIG
    assert b"at least 2 clusters" in lib.rv_last_error()
    rl2 = (ctypes.c_int64 * 1)(9)
    assert lib.rv_plan_create(ctypes.byref(h), 0, 2, 1, rs, rl2, 10, 0, 0) == _native.RV_E_LAYOUT
    assert lib.rv_plan_create(ctypes.byref(h), 0, 2, 1, rs, rl, 10, 7, 0) == _native.RV_E_CONFIG


@pytest.mark.parametrize("lens", [[10], [5, 0, 7, 100], [26201088, 27168768, 27170304, 28942080], [3] * 9, [0, 0]])
@pytest.mark.parametrize("n_lanes", [1, 2, 3, 4, 9, 16, 64])
def test_lane_partition(lens, n_lanes):
    # lanes tile [0, total) in order; up to R lanes they are unions of whole
    # rings (R lanes = one ring each), beyond R they never straddle a ring
    starts = [sum(lens[:i]) for i in range(len(lens))]
    total = sum(lens)
    R = len(lens)
    if n_lanes > max(64, R):
        pytest.skip("beyond capacity")
    got = _native.lane_ranges(starts, lens, n_lanes)
    assert len(got) == n_lanes
    cursor = 0
    for lo, hi in got:
        assert lo == cursor and hi >= lo
        cursor = hi
    assert cursor == total
    edges = set(starts) | {total}
    if n_lanes <= R:
        assert all(lo in edges and hi in edges for lo, hi in got)
        if n_lanes == R:
            assert got == [(s, s + n) for s, n in zip(starts, lens)]
    else:
        for lo, hi in got:
            if hi > lo:
                r = max(i for i, s in enumerate(starts) if s <= lo)
                assert hi <= starts[r] + lens[r]


def test_plan_option_ids_match_the_header():
    """rv_plan_set_option's RV_OPT_* ids in the header are the ones the
    Python plans pass (kernel choice comes only from these, never from the
    environment)."""
    with open(os.path.join(ROOT, "include", "ravnest_b200.h")) as f:
        defs = dict((k, int(v)) for k, v in re.findall(r"^#define (RV_OPT_\w+) (\d+)", f.read(), re.M))
    assert defs == {f"RV_OPT_{k.upper()}": v for k, v in _native.OPTIONS.items()}
    src = open(os.path.join(ROOT, "paper_2401_01728_b200", "csrc", "ravnest_b200.cu")).read()
    src += open(os.path.join(ROOT, "paper_2401_01728_b200", "csrc", "rv_dispatch.cuh")).read()
    assert "getenv" not in src
