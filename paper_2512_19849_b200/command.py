"""TransferCmd: the 16-byte GPU->CPU control word (drop-in for epsim.command).

Same names, fields, bit layout and error behaviour as command.py:1-158; the
work is done by the C ABI (codec.cpp), which is also what the CUDA producer
(ll.cu) and the C++ proxy (proxy.cpp) use, so a command packed anywhere
decodes identically everywhere.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

import ctypes as C

from ._lib import check, lib, nptr

from .errors import ProtocolViolation

WRITE, ATOMIC, DRAIN, BARRIER = 0, 1, 2, 3
KIND_NAMES = {WRITE: "Write", ATOMIC: "Atomic", DRAIN: "Drain", BARRIER: "Barrier"}
FLAG_PIGGYBACK_ATOMIC = 1
FLAG_SAME_RAIL_BARRIER = 2
CMD_BYTES = 16


@dataclass(frozen=True)
class TransferCmd:
    kind: int
    dst_rank: int = 0
    channel_id: int = 0
    src_offset: int = 0
    dst_offset: int = 0
    length_or_value: int = 0
    flags: int = 0

    def validate(self) -> None:
        pack(self)


def pack(cmd: TransferCmd) -> tuple[int, int]:
    lo, hi = C.c_uint64(), C.c_uint64()
    fields = (cmd.kind, cmd.dst_rank, cmd.channel_id, cmd.src_offset, cmd.dst_offset, cmd.length_or_value, cmd.flags)
    if any(not -(1 << 63) <= f < (1 << 63) for f in fields):
        raise ProtocolViolation("field out of range")
    check(lib.epb_cmd_pack(*fields, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def unpack(lo: int, hi: int) -> TransferCmd:
    f = unpack_fields(np.array([lo & (2**64 - 1)], np.uint64), np.array([hi & (2**64 - 1)], np.uint64))
    return TransferCmd(**{k: int(v[0]) for k, v in f.items()})


def to_bytes(cmd: TransferCmd) -> bytes:
    return struct.pack("<QQ", *pack(cmd))


def from_bytes(raw: bytes) -> TransferCmd:
    if len(raw) != CMD_BYTES:
        raise ProtocolViolation(f"command record must be {CMD_BYTES} bytes, got {len(raw)}")
    return unpack(*struct.unpack("<QQ", raw))


_FIELDS = ("kind", "dst_rank", "channel_id", "src_offset", "dst_offset", "length_or_value", "flags")


def pack_fields(kind, dst_rank, channel_id, src_offset, dst_offset, length_or_value, flags):
    arrs = [np.ascontiguousarray(np.asarray(a).astype(np.uint64).view(np.int64)).ravel()
            for a in (kind, dst_rank, channel_id, src_offset, dst_offset, length_or_value, flags)]
    n = max(len(a) for a in arrs)
    arrs = [np.broadcast_to(a, (n,)).copy() if len(a) != n else a for a in arrs]
    lo = np.empty(n, np.uint64)
    hi = np.empty(n, np.uint64)
    check(lib.epb_cmd_pack_fields(*[nptr(a, C.c_int64) for a in arrs], n, nptr(lo, C.c_uint64), nptr(hi, C.c_uint64)))
    return lo, hi


def unpack_fields(lo, hi) -> dict:
    lo = np.ascontiguousarray(np.asarray(lo).astype(np.uint64)).ravel()
    hi = np.ascontiguousarray(np.asarray(hi).astype(np.uint64)).ravel()
    n = len(lo)
    outs = {k: np.empty(n, np.int64) for k in _FIELDS}
    check(lib.epb_cmd_unpack_fields(nptr(lo, C.c_uint64), nptr(hi, C.c_uint64), n,
                                    *[nptr(outs[k], C.c_int64) for k in _FIELDS]))
    return outs


__all__ = ["TransferCmd", "pack", "unpack", "to_bytes", "from_bytes", "pack_fields", "unpack_fields", "WRITE",
           "ATOMIC", "DRAIN", "BARRIER", "FLAG_PIGGYBACK_ATOMIC", "FLAG_SAME_RAIL_BARRIER", "CMD_BYTES"]
