"""Byte formats next to the averaging path.

* Session plans: read the ``[layouts]``/``[rings]``/``[pipelines]`` sections
  of a ``ravnest-plan-v1`` file written by the reference's
  ``configio.serialize_plan`` (configio.py:147-173, parsed at :226-246), so a
  plan formed by the reference CLI drives the GPU cycle directly; and write
  the ``[rings]`` rows back (``ring_id start len cid:peer,...``).
* Wire frames for a multi-box transport (multiring.py:398-426):
  ``u32 length | u8 kind | u32 ring_id | u32 round | u64 offset | fp64[]``,
  little-endian, bit-exact with the reference.
* Checkpoints (configio.py:495-512): ``b"RAVNCKPT" | u32 version | u64 count |
  count x fp64 LE``; ``save_device_checkpoint`` widens on the GPU and copies
  the averaged parameters to the host once.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ProtocolError, SchemaError
from .schedule import ParamRange, Ring, RingSchedule, chunk_bounds, validate_schedule

PLAN_SCHEMA = "ravnest-plan-v1"
CHECKPOINT_MAGIC = b"RAVNCKPT"
CHECKPOINT_VERSION = 1
FRAME_KIND_CODES = {"control": 0, "activation": 1, "gradient": 2, "ring_chunk": 3}
_FRAME_KINDS = {v: k for k, v in FRAME_KIND_CODES.items()}
_HEAD = struct.Struct("<BIIQ")
_LEN = struct.Struct("<I")
_CKPT_HEAD = struct.Struct("<IQ")


# ---------------------------------------------------------------------------
# session plans


@dataclass
class PlanRings:
    """What the averaging path needs from a session plan."""

    schedule: RingSchedule
    layouts: dict[int, list[ParamRange]]
    pipelines: dict[int, list[str]]

    @property
    def cluster_ids(self) -> list[int]:
        return sorted(self.layouts)

    def node_of(self, cluster_id: int, peer: int) -> str:
        return self.pipelines[cluster_id][peer]


def _sections(text: str) -> dict[str, list[str]]:
    secs: dict[str, list[str]] = {}
    cur = None
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line[0] == "[" and line[-1] == "]":
            cur = line[1:-1].strip()
            secs.setdefault(cur, [])
        elif cur is None:
            raise SchemaError(f"content before any section header: {line!r}")
        else:
            secs[cur].append(line)
    return secs


def read_plan(text: str) -> PlanRings:
    """Ring schedule, per-cluster submodel spans and node names of a plan."""
    lines = text.splitlines()
    head = lines[0].strip() if lines else ""
    if head != f"# schema: {PLAN_SCHEMA}":
        raise SchemaError(f"not a {PLAN_SCHEMA} file (got {head!r})")
    secs = _sections(text)
    for need in ("layouts", "rings", "pipelines"):
        if need not in secs:
            raise SchemaError(f"plan has no [{need}] section")
    pipelines = {}
    for row in secs["pipelines"]:
        cid, *nodes = row.split()
        pipelines[int(cid)] = nodes
    layouts: dict[int, list[ParamRange]] = {}
    for row in secs["layouts"]:
        f = row.split()
        if len(f) != 6:
            raise SchemaError(f"layout row needs 6 fields: {row!r}")
        cid, peer, start, length = int(f[0]), int(f[1]), int(f[4]), int(f[5])
        lay = layouts.setdefault(cid, [])
        if len(lay) != peer:
            raise SchemaError(f"layout rows for cluster {cid} out of order")
        lay.append(ParamRange(start, length))
    rings = []
    for row in secs["rings"]:
        f = row.split()
        if len(f) != 4:
            raise SchemaError(f"ring row needs 4 fields: {row!r}")
        members = tuple(tuple(int(v) for v in m.split(":")) for m in f[3].split(","))
        rings.append(Ring(int(f[0]), int(f[1]), int(f[2]), members))
    total = max((s.param_start + s.param_len for lay in layouts.values() for s in lay), default=0)
    schedule = RingSchedule(tuple(rings), total)
    validate_schedule(schedule, layouts)
    return PlanRings(schedule, layouts, pipelines)


def read_plan_file(path: str | Path) -> PlanRings:
    return read_plan(Path(path).read_text())


def rings_section(schedule) -> str:
    """The ``[rings]`` section of a plan file for ``schedule``."""
    out = ["[rings]"]
    for r in schedule.rings:
        out.append(f"{r.ring_id} {r.start} {r.length} " + ",".join(f"{c}:{p}" for c, p in r.members))
    return "\n".join(out) + "\n"


# ---------------------------------------------------------------------------
# wire frames


def encode_frame(kind: str, ring_id: int, round_idx: int, offset: int, payload) -> bytes:
    if kind not in FRAME_KIND_CODES:
        raise ProtocolError(f"unknown frame kind {kind!r}")
    body = _HEAD.pack(FRAME_KIND_CODES[kind], ring_id, round_idx, offset)
    body += np.ascontiguousarray(payload, dtype="<f8").tobytes()
    return _LEN.pack(len(body)) + body


def decode_frame(buf: bytes) -> tuple[str, int, int, int, np.ndarray, int]:
    """Fields of the first frame in ``buf`` plus the bytes it used."""
    if len(buf) < _LEN.size:
        raise ProtocolError("frame shorter than its length prefix")
    (n,) = _LEN.unpack_from(buf, 0)
    if len(buf) < _LEN.size + n:
        raise ProtocolError(f"truncated frame: need {n} body bytes")
    code, ring_id, round_idx, offset = _HEAD.unpack_from(buf, _LEN.size)
    if code not in _FRAME_KINDS:
        raise ProtocolError(f"unknown frame kind code {code}")
    count = (n - _HEAD.size) // 8
    payload = np.frombuffer(buf, dtype="<f8", count=count, offset=_LEN.size + _HEAD.size).copy()
    return _FRAME_KINDS[code], ring_id, round_idx, offset, payload, _LEN.size + n


def owner_chunk_frames(schedule, values, position: int, n_clusters: int) -> list[bytes]:
    """One ``ring_chunk`` frame per ring carrying chunk ``position`` of
    ``values`` (host array or CUDA tensor), tagged with the last round of the
    cycle -- what the owner of that chunk would put on a wire to a remote box."""
    if hasattr(values, "is_cuda") and values.is_cuda:
        values = values.double().cpu().numpy()
    values = np.asarray(values)
    last_round = 2 * (n_clusters - 1) - 1
    out = []
    for r in schedule.rings:
        lo, hi = chunk_bounds(r.start, r.length, n_clusters)[position]
        out.append(encode_frame("ring_chunk", r.ring_id, last_round, lo, values[lo:hi]))
    return out


# ---------------------------------------------------------------------------
# checkpoints


def write_checkpoint(path: str | Path, values) -> None:
    arr = np.ascontiguousarray(values, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(CHECKPOINT_MAGIC)
        fh.write(_CKPT_HEAD.pack(CHECKPOINT_VERSION, arr.size))
        fh.write(arr.tobytes())


def read_checkpoint(path: str | Path) -> np.ndarray:
    raw = Path(path).read_bytes()
    if raw[:8] != CHECKPOINT_MAGIC:
        raise SchemaError(f"{path}: not a ravnest checkpoint")
    version, count = _CKPT_HEAD.unpack_from(raw, 8)
    if version != CHECKPOINT_VERSION:
        raise SchemaError(f"{path}: unsupported checkpoint version {version}")
    return np.frombuffer(raw, dtype="<f8", count=count, offset=8 + _CKPT_HEAD.size).astype(np.float64)


def save_device_checkpoint(path: str | Path, tensor) -> None:
    """Checkpoint an averaged parameter vector straight from the GPU (the
    float64 widening runs on the device; one D2H copy)."""
    write_checkpoint(path, tensor.detach().reshape(-1).double().cpu().numpy())
