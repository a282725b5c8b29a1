"""Device plans and single-process ring groups.

``DevicePlan`` owns one ``rv_plan`` (include/ravnest_b200.h): the chunk
tables, lane state and barrier flags of one GPU.  ``LocalRingGroup`` places
C clusters on one or more GPUs of this process -- all on one GPU is the
co-resident case (no barriers), one per GPU uses NVLink peer access with
device-side flags.  The multi-process (one process per GPU) group is
``dist.DistRingGroup``.

Reference seam: the per-cycle call is what ``orchestrator._maybe_average``
(orchestrator.py:320-337) makes through ``multiring.apply_ring_mean``.
"""

from __future__ import annotations

import ctypes
import os
from typing import Iterable, Mapping, Sequence

from . import _native as N
from .errors import ConfigError, LayoutError

ACC_MODES = {"f64": N.RV_ACC_F64, "native": N.RV_ACC_NATIVE}
PROTOCOLS = {"pull": N.RV_PROTO_PULL, "push": N.RV_PROTO_PUSH, "ll": N.RV_PROTO_LL}


def _dtype_code(dtype) -> int:
    name = str(dtype)
    if name.endswith("float32"):
        return N.RV_DTYPE_F32
    if name.endswith("float64"):
        return N.RV_DTYPE_F64
    raise ConfigError(f"unsupported parameter dtype {dtype} (float32 or float64)")


def _stream_handle(stream) -> int:
    if stream is None:
        return 0
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


class DevicePlan:
    """One rv_plan: the slice of a cycle that runs on ``device``."""

    def __init__(self, device: int, n_clusters: int, starts: Sequence[int], lens: Sequence[int],
                 total: int, dtype_code: int, acc: str = "f64"):
        if acc not in ACC_MODES:
            raise ConfigError(f"unknown accumulation mode {acc!r} (use 'f64' or 'native')")
        self.lib = N.load()
        self.device = int(device)
        self.n_clusters = int(n_clusters)
        self.n_rings = len(starts)
        rs = (ctypes.c_int64 * max(1, len(starts)))(*[int(s) for s in starts])
        rl = (ctypes.c_int64 * max(1, len(lens)))(*[int(n) for n in lens])
        h = ctypes.c_void_p()
        N.check(self.lib.rv_plan_create(ctypes.byref(h), self.device, self.n_clusters, len(starts), rs, rl,
                                        int(total), int(dtype_code), ACC_MODES[acc]), "rv_plan_create")
        self._h = h
        self._launch = self.lib.rv_allreduce_mean
        self._stream_cache: dict = {}
        timeout = os.environ.get("RAVNEST_B200_TIMEOUT_S")  # deployment setting, not a kernel choice
        if timeout and float(timeout) > 0:
            self.set_timeout(float(timeout))

    @property
    def handle(self):
        return self._h

    def bind(self, pos: int, src_ptr: int, dst_ptr: int) -> None:
        N.check(self.lib.rv_plan_bind(self._h, int(pos), ctypes.c_void_p(int(src_ptr)),
                                      ctypes.c_void_p(int(dst_ptr))), "rv_plan_bind")

    def bind_live(self, pos: int, live_ptr: int | None) -> None:
        """Blend target of position ``pos`` (``None`` unbinds): every cycle
        then also leaves live <- mean + (live - src) there."""
        N.check(self.lib.rv_plan_bind_live(self._h, int(pos), ctypes.c_void_p(int(live_ptr or 0))),
                "rv_plan_bind_live")

    def set_local(self, positions: Iterable[int]) -> None:
        pos = [int(p) for p in positions]
        arr = (ctypes.c_int * max(1, len(pos)))(*pos)
        N.check(self.lib.rv_plan_set_local(self._h, arr, len(pos)), "rv_plan_set_local")

    def set_lanes(self, n: int) -> None:
        N.check(self.lib.rv_plan_set_lanes(self._h, int(n)), "rv_plan_set_lanes")

    def set_protocol(self, proto: str) -> None:
        if proto not in PROTOCOLS:
            raise ConfigError(f"unknown protocol {proto!r} (use 'pull', 'push' or 'll')")
        N.check(self.lib.rv_plan_set_protocol(self._h, PROTOCOLS[proto]), "rv_plan_set_protocol")

    def push_area(self) -> tuple[int, int]:
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        N.check(self.lib.rv_plan_push_area(self._h, ctypes.byref(p), ctypes.byref(n)), "rv_plan_push_area")
        return int(p.value or 0), int(n.value)

    def set_push_peers(self, areas: Sequence[int]) -> None:
        N.check(self.lib.rv_plan_set_push_peers(self._h, N.ptr_array(areas)), "rv_plan_set_push_peers")

    def set_option(self, name: str, value: int) -> None:
        """rv_plan_set_option: ``min_cb``, ``tma``, ``push_items``, ``push_dyn``,
        ``blend_lag``, ``layout_sms`` (include/ravnest_b200.h RV_OPT_*)."""
        if name not in N.OPTIONS:
            raise ConfigError(f"unknown plan option {name!r} (one of {sorted(N.OPTIONS)})")
        N.check(self.lib.rv_plan_set_option(self._h, N.OPTIONS[name], int(value)), f"rv_plan_set_option({name})")

    def set_options(self, options: Mapping[str, int] | None) -> None:
        for name, value in (options or {}).items():
            self.set_option(name, value)

    def prepare(self) -> None:
        """Build the device tables now (every position bound)."""
        N.check(self.lib.rv_plan_prepare(self._h), "rv_plan_prepare")

    def layout(self) -> tuple[int, int, int, int]:
        """(vectors per unit, staging stride, unit slots, work items per lane)
        of the built tables; push / LL ranks must agree on it."""
        out = (ctypes.c_int64 * 4)()
        N.check(self.lib.rv_plan_layout(self._h, out), "rv_plan_layout")
        return tuple(int(v) for v in out)

    def failed(self) -> bool:
        """Non-blocking: a cycle of this plan hit its stall timeout."""
        return bool(self.lib.rv_plan_failed(self._h))

    def set_max_blocks(self, n: int) -> None:
        N.check(self.lib.rv_plan_set_max_blocks(self._h, int(n)), "rv_plan_set_max_blocks")

    def set_trace(self, enable: bool = True) -> None:
        N.check(self.lib.rv_plan_set_trace(self._h, int(bool(enable))), "rv_plan_set_trace")

    def read_trace(self, lane: int = 0) -> dict:
        """Phase durations (us) of the last launch of `lane`: launch->ready
        (pull: arrive barrier), ready->data done, data done->departed."""
        out = (ctypes.c_uint64 * 4)()
        N.check(self.lib.rv_plan_read_trace(self._h, int(lane), out), "rv_plan_read_trace")
        t0, t1, t2, t3 = (int(v) for v in out)
        t3 = t3 or t2
        return {"ready_us": (t1 - t0) / 1e3, "data_us": (t2 - t1) / 1e3, "depart_us": (t3 - t2) / 1e3,
                "total_us": (t3 - t0) / 1e3}

    def set_timeout(self, seconds: float) -> None:
        N.check(self.lib.rv_plan_set_timeout(self._h, float(seconds)), "rv_plan_set_timeout")

    def flag_area(self) -> tuple[int, int]:
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        N.check(self.lib.rv_plan_flag_area(self._h, ctypes.byref(p), ctypes.byref(n)), "rv_plan_flag_area")
        return int(p.value or 0), int(n.value)

    def set_peers(self, rank: int, n_ranks: int, areas: Sequence[int]) -> None:
        arr = N.ptr_array(areas)
        N.check(self.lib.rv_plan_set_peers(self._h, int(rank), int(n_ranks), arr), "rv_plan_set_peers")

    def run(self, streams: Sequence = (None,)) -> None:
        key = tuple(_stream_handle(s) for s in streams) or (0,)
        arr = self._stream_cache.get(key)
        if arr is None:  # ctypes arrays are cached: the launch path stays a few microseconds
            arr = self._stream_cache[key] = N.ptr_array(key)
        rc = self._launch(self._h, arr, len(key))
        if rc:
            N.check(rc, "rv_allreduce_mean")

    def run_lanes(self, first: int, count: int, streams: Sequence = (None,)) -> None:
        key = tuple(_stream_handle(s) for s in streams) or (0,)
        arr = self._stream_cache.get(key)
        if arr is None:
            arr = self._stream_cache[key] = N.ptr_array(key)
        N.check(self.lib.rv_allreduce_mean_lanes(self._h, int(first), int(count), arr, len(key)),
                "rv_allreduce_mean_lanes")

    def run_host(self, host_src: Sequence[int], host_dst: Sequence[int], streams: Sequence = (None,)) -> None:
        hs = [_stream_handle(s) for s in streams] or [0]
        N.check(self.lib.rv_allreduce_mean_host(self._h, N.ptr_array(host_src), N.ptr_array(host_dst),
                                                N.ptr_array(hs), len(hs)), "rv_allreduce_mean_host")

    def run_host_lanes(self, first: int, count: int, host_src: Sequence[int], host_dst: Sequence[int],
                       streams: Sequence = (None,)) -> None:
        hs = [_stream_handle(s) for s in streams] or [0]
        N.check(self.lib.rv_allreduce_mean_host_lanes(self._h, int(first), int(count), N.ptr_array(host_src),
                                                      N.ptr_array(host_dst), N.ptr_array(hs), len(hs)),
                "rv_allreduce_mean_host_lanes")

    def status(self) -> tuple[int, str]:
        buf = ctypes.create_string_buffer(512)
        rc = self.lib.rv_plan_status(self._h, buf, len(buf))
        return rc, buf.value.decode(errors="replace")

    def check_status(self) -> None:
        rc, diag = self.status()
        if rc != N.RV_OK:
            N.check(rc, diag)

    def reset_status(self) -> None:
        N.check(self.lib.rv_plan_reset_status(self._h), "rv_plan_reset_status")

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.rv_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class LocalRingGroup:
    """C clusters placed on GPUs of this process (position m on ``devices[m]``).

    Position m is the m-th smallest cluster id (ring member order,
    multiring.py:95).  One DevicePlan per distinct device; each folds the
    chunks of the positions it hosts.  With more than one device the plans
    meet through device-side flags over NVLink peer access.
    """

    def __init__(self, starts: Sequence[int], lens: Sequence[int], total: int, devices: Sequence[int],
                 dtype, acc: str = "f64", lanes: int = 1, protocol: str = "pull",
                 options: Mapping[str, int] | None = None):
        self.starts = [int(s) for s in starts]
        self.lens = [int(n) for n in lens]
        self.total = int(total)
        self.devices = [int(d) for d in devices]
        self.n_clusters = len(self.devices)
        if self.n_clusters < 2:
            raise ConfigError("all-reduce needs at least 2 clusters")
        self.dtype_code = _dtype_code(dtype)
        self.acc = acc
        self.device_order = sorted(set(self.devices))
        lib = N.load()
        if len(self.device_order) > 1:
            for a in self.device_order:
                for b in self.device_order:
                    if a != b:
                        N.check(lib.rv_enable_peer_access(a, b), "rv_enable_peer_access")
        self.plans: dict[int, DevicePlan] = {}
        for d in self.device_order:
            plan = DevicePlan(d, self.n_clusters, self.starts, self.lens, self.total, self.dtype_code, acc)
            plan.set_local([m for m, dev in enumerate(self.devices) if dev == d])
            plan.set_options(options)
            if lanes != 1:
                plan.set_lanes(lanes)
            self.plans[d] = plan
        if len(self.device_order) > 1:
            areas = [self.plans[d].flag_area()[0] for d in self.device_order]
            for rank, d in enumerate(self.device_order):
                self.plans[d].set_peers(rank, len(self.device_order), areas)
        self.protocol = protocol if len(self.device_order) > 1 else "pull"
        if self.protocol in ("push", "ll"):
            # owner-staged transports: one cluster per device, position == rank
            if sorted(self.devices) != self.devices or len(set(self.devices)) != len(self.devices):
                raise ConfigError(f"{self.protocol} needs one cluster per device, in device order")
            push = []
            for d in self.device_order:
                self.plans[d].set_protocol(self.protocol)
                push.append(self.plans[d].push_area()[0])
            for d in self.device_order:
                self.plans[d].set_push_peers(push)
        elif self.protocol != "pull":
            raise ConfigError(f"unknown protocol {protocol!r}")

    def bind(self, pos: int, src_ptr: int, dst_ptr: int) -> None:
        for plan in self.plans.values():
            plan.bind(pos, src_ptr, dst_ptr)

    def bind_tensors(self, srcs: Sequence, dsts: Sequence | None = None) -> None:
        dsts = srcs if dsts is None else dsts
        for m, (s, d) in enumerate(zip(srcs, dsts)):
            if s.device.index != self.devices[m] or d.device.index != self.devices[m]:
                raise LayoutError(f"cluster position {m} tensor is on {s.device}, plan expects cuda:{self.devices[m]}")
            if s.numel() != self.total or d.numel() != self.total:
                raise LayoutError(f"cluster position {m} vector has {s.numel()} elements, schedule expects {self.total}")
            if not (s.is_contiguous() and d.is_contiguous()):
                raise LayoutError(f"cluster position {m} tensor must be contiguous")
            self.bind(m, s.data_ptr(), d.data_ptr())
        self._bound = (list(srcs), list(dsts))  # the plans hold raw pointers: keep the tensors alive

    def bind_live(self, lives: Sequence | None) -> None:
        """Delayed-update blend fused into the cycle: ``lives[m]`` (a tensor
        like position m's src) ends every cycle as mean + (live - src).
        Needs separate src and dst buffers.  ``None`` unbinds."""
        for m in range(self.n_clusters):
            ptr = None
            if lives is not None:
                t = lives[m]
                if t.device.index != self.devices[m] or t.numel() != self.total or not t.is_contiguous():
                    raise LayoutError(f"live tensor of position {m} does not match its cluster vector")
                ptr = t.data_ptr()
            for d, plan in self.plans.items():
                if d == self.devices[m]:
                    plan.bind_live(m, ptr)
        self._lives = None if lives is None else list(lives)

    def run(self, streams: dict | None = None) -> None:
        """Launch one cycle.  ``streams`` maps device -> stream (or a list of
        streams for per-ring lanes); default is torch's current stream."""
        import torch

        with torch.cuda.nvtx.range("ravnest_b200.cycle"):
            self._run(streams)

    def _run(self, streams) -> None:
        import torch

        for d in self.device_order:
            if streams is not None and d in streams:
                st = streams[d]
                st = st if isinstance(st, (list, tuple)) else [st]
            else:
                st = [torch.cuda.current_stream(d)]
            self.plans[d].run(st)

    def check(self) -> None:
        for plan in self.plans.values():
            plan.check_status()

    def failed(self) -> bool:
        """Non-blocking: a cycle of one of the plans stalled."""
        return any(plan.failed() for plan in self.plans.values())

    def close(self) -> None:
        for plan in self.plans.values():
            plan.close()
        self.plans = {}
        # drop the buffers kept alive for the plans (and the numpy drop-in's
        # device staging, multiring._HostCycle) so an evicted group frees them
        for attr in ("_bound", "_lives", "_host_bufs", "_host_streams"):
            if hasattr(self, attr):
                setattr(self, attr, None)
