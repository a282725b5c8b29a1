"""ctypes binding of libravnest_b200.so (the C ABI in include/ravnest_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of the compute entry points raises, loudly.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, LayoutError, RavnestError, StallError

LIB_NAME = "libravnest_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

RV_OK = 0
RV_E_CONFIG = 1
RV_E_LAYOUT = 2
RV_E_CUDA = 3
RV_E_PEER_ACCESS = 4
RV_E_TIMEOUT = 5
RV_E_ARG = 6

RV_DTYPE_F32 = 0
RV_DTYPE_F64 = 1
RV_ACC_F64 = 0
RV_ACC_NATIVE = 1

RV_PROTO_PULL = 0
RV_PROTO_PUSH = 1
RV_PROTO_LL = 2

RV_OPT_MIN_CB = 1
RV_OPT_TMA = 2
RV_OPT_PUSH_ITEMS = 3
RV_OPT_PUSH_DYN = 4
RV_OPT_BLEND_LAG = 5
RV_OPT_LAYOUT_SMS = 6
OPTIONS = {"min_cb": RV_OPT_MIN_CB, "tma": RV_OPT_TMA, "push_items": RV_OPT_PUSH_ITEMS,
           "push_dyn": RV_OPT_PUSH_DYN, "blend_lag": RV_OPT_BLEND_LAG, "layout_sms": RV_OPT_LAYOUT_SMS}

RV_MAX_CLUSTERS = 16
RV_MAX_RANKS = 16

_c_void_pp = ctypes.POINTER(ctypes.c_void_p)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); every symbol include/ravnest_b200.h declares
SIGNATURES = {
    "rv_version": (ctypes.c_int, []),
    "rv_last_error": (ctypes.c_char_p, []),
    "rv_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "rv_plan_create": (ctypes.c_int, [_c_void_pp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i64_p, _c_i64_p,
                                      ctypes.c_int64, ctypes.c_int, ctypes.c_int]),
    "rv_plan_bind": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "rv_plan_bind_live": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "rv_plan_set_local": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_int]),
    "rv_plan_set_lanes": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rv_lane_ranges": (ctypes.c_int, [ctypes.c_int, _c_i64_p, _c_i64_p, ctypes.c_int, _c_i64_p, _c_i64_p]),
    "rv_plan_flag_area": (ctypes.c_int, [ctypes.c_void_p, _c_void_pp, ctypes.POINTER(ctypes.c_size_t)]),
    "rv_plan_set_peers": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _c_void_pp]),
    "rv_plan_set_protocol": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rv_plan_push_area": (ctypes.c_int, [ctypes.c_void_p, _c_void_pp, ctypes.POINTER(ctypes.c_size_t)]),
    "rv_plan_set_push_peers": (ctypes.c_int, [ctypes.c_void_p, _c_void_pp]),
    "rv_plan_set_timeout": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double]),
    "rv_plan_set_option": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64]),
    "rv_plan_prepare": (ctypes.c_int, [ctypes.c_void_p]),
    "rv_plan_layout": (ctypes.c_int, [ctypes.c_void_p, _c_i64_p]),
    "rv_plan_failed": (ctypes.c_int, [ctypes.c_void_p]),
    "rv_plan_set_trace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rv_plan_set_max_blocks": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "rv_plan_read_trace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]),
    "rv_allreduce_mean": (ctypes.c_int, [ctypes.c_void_p, _c_void_pp, ctypes.c_int]),
    "rv_allreduce_mean_lanes": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _c_void_pp, ctypes.c_int]),
    "rv_allreduce_mean_host": (ctypes.c_int, [ctypes.c_void_p, _c_void_pp, _c_void_pp, _c_void_pp, ctypes.c_int]),
    "rv_allreduce_mean_host_lanes": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _c_void_pp, _c_void_pp,
                                                    _c_void_pp, ctypes.c_int]),
    "rv_plan_status": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]),
    "rv_plan_reset_status": (ctypes.c_int, [ctypes.c_void_p]),
    "rv_plan_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "rv_blend": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.c_void_p]),
    "rv_ipc_handle_size": (ctypes.c_int, []),
    "rv_ipc_export": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]),
    "rv_ipc_import": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, _c_void_pp]),
    "rv_ipc_close": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p]),
    "rv_enable_peer_access": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "rv_device_sm_count": (ctypes.c_int, [ctypes.c_int]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the CUDA library; raise if it is absent (no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RavnestError(
            f"{LIB_NAME} not found at {LIB_PATH}: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.rv_version() != 1:
        raise RavnestError(f"{LIB_NAME} ABI version {lib.rv_version()} != 1")
    _lib = lib
    return lib


def last_error() -> str:
    return load().rv_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map C status codes onto the reference's exception classes (errors.py:4-65)."""
    if rc == RV_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == RV_E_CONFIG:
        raise ConfigError(msg)
    if rc == RV_E_LAYOUT:
        raise LayoutError(msg)
    if rc == RV_E_TIMEOUT:
        raise StallError(msg)
    raise RavnestError(msg)


def ptr_array(ptrs) -> ctypes.Array:
    return (ctypes.c_void_p * max(1, len(ptrs)))(*[ctypes.c_void_p(int(p)) for p in ptrs])


def lane_ranges(starts, lens, n_lanes: int) -> list[tuple[int, int]]:
    """The element ranges the C plan assigns to its lanes (rv_lane_ranges)."""
    lib = load()
    R = len(lens)
    rs = (ctypes.c_int64 * max(1, R))(*[int(x) for x in starts])
    rl = (ctypes.c_int64 * max(1, R))(*[int(x) for x in lens])
    lo = (ctypes.c_int64 * n_lanes)()
    hi = (ctypes.c_int64 * n_lanes)()
    check(lib.rv_lane_ranges(R, rs, rl, int(n_lanes), lo, hi), "rv_lane_ranges")
    return list(zip(lo, hi))
