"""ctypes wrapper over oracle/_build/libring_oracle.so -- TEST INFRASTRUCTURE ONLY.

See ring_oracle.c for what it restates.  Importable only from tests/,
__graft_entry__.smoke() and bench.py's CPU legs.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libring_oracle.so")

MODE_F64 = 0
MODE_F32_ACC64 = 1
MODE_F32_NATIVE = 2

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.rvo_ring_mean.restype = ctypes.c_int
        lib.rvo_ring_mean.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
            ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
            ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
        ]
        _lib = lib
    return _lib


def _ptrs(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def ring_mean_into(mode: int, ring_starts, ring_lens, inputs: Sequence[np.ndarray],
                   outputs: Sequence[np.ndarray] | None, outputs32: Sequence[np.ndarray] | None = None,
                   threads: int = 1) -> None:
    lib = _load()
    c = len(inputs)
    rs = np.ascontiguousarray(ring_starts, dtype=np.int64)
    rl = np.ascontiguousarray(ring_lens, dtype=np.int64)
    out_p = _ptrs(outputs) if outputs is not None else None
    out32_p = _ptrs(outputs32) if outputs32 is not None else None
    rc = lib.rvo_ring_mean(
        mode, c, len(rs),
        rs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        rl.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        _ptrs(inputs), out_p, out32_p, int(threads),
    )
    if rc != 0:
        raise RuntimeError("rvo_ring_mean failed")


def ring_mean(ring_starts, ring_lens, inputs: Sequence[np.ndarray], mode: int = MODE_F64,
              threads: int = 1) -> list[np.ndarray]:
    """Returns new arrays (f64 for MODE_F64/MODE_F32_ACC64, f32 for native)."""
    if mode == MODE_F64:
        ins = [np.ascontiguousarray(v, dtype=np.float64) for v in inputs]
        outs = [v.copy() for v in ins]
    elif mode == MODE_F32_ACC64:
        ins = [np.ascontiguousarray(v, dtype=np.float32) for v in inputs]
        outs = [v.astype(np.float64) for v in ins]
    else:
        ins = [np.ascontiguousarray(v, dtype=np.float32) for v in inputs]
        outs = [v.copy() for v in ins]
    ring_mean_into(mode, ring_starts, ring_lens, ins, outs, None, threads)
    return outs
