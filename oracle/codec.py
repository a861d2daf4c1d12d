"""Oracle restatement of the TransferCmd and immediate-word codecs.

Follows command.py:8-13 (bit layout), command.py:55-67 (validate),
command.py:70-97 (pack/unpack), command.py:100-110 (16-byte LE records),
command.py:113-158 (vectorised), and imm.py:7-91.  Pinned by
tests/test_oracle_golden.py against vectors produced by the reference.
"""
from __future__ import annotations

import struct

import numpy as np

WRITE, ATOMIC, DRAIN, BARRIER = 0, 1, 2, 3
FLAG_PIGGYBACK_ATOMIC, FLAG_SAME_RAIL_BARRIER = 1, 2
U64 = np.uint64


class CodecError(ValueError):
    pass


def _check(kind, dst_rank, channel_id, src_offset, dst_offset, length_or_value, flags):  # command.py:55-67
    if not 0 <= kind <= 3:
        raise CodecError("kind")
    if not 0 <= dst_rank < (1 << 12):
        raise CodecError("dst_rank")
    if not 0 <= channel_id < (1 << 6):
        raise CodecError("channel_id")
    for v in (src_offset, dst_offset, length_or_value):
        if not 0 <= v < (1 << 32):
            raise CodecError("u32 field")
    if not 0 <= flags <= 3:
        raise CodecError("flags")


def pack(kind, dst_rank=0, channel_id=0, src_offset=0, dst_offset=0, length_or_value=0, flags=0):
    """command.py:70-81: returns (lo, hi) Python ints."""
    _check(kind, dst_rank, channel_id, src_offset, dst_offset, length_or_value, flags)
    lo = kind + (dst_rank << 2) + (channel_id << 14) + (src_offset << 20) + ((dst_offset % 4096) << 52)
    hi = (dst_offset >> 12) + (length_or_value << 20) + (flags << 52)
    return lo, hi


def unpack(lo, hi):
    """command.py:84-97: returns the 7 fields as a tuple."""
    lo %= 1 << 64
    hi %= 1 << 64
    if hi >> 54:
        raise CodecError("reserved bits")
    return (lo % 4, (lo >> 2) % 4096, (lo >> 14) % 64, (lo >> 20) % (1 << 32),
            ((lo >> 52) + ((hi % (1 << 20)) << 12)) % (1 << 32), (hi >> 20) % (1 << 32), (hi >> 52) % 4)


def to_bytes(lo, hi) -> bytes:  # command.py:100-104
    return struct.pack("<QQ", lo, hi)


def pack_fields(kind, dst_rank, channel_id, src_offset, dst_offset, length_or_value, flags):
    """command.py:113-138 (unvalidated, uint64 arithmetic)."""
    f = [np.asarray(a).astype(U64) for a in (kind, dst_rank, channel_id, src_offset, dst_offset,
                                             length_or_value, flags)]
    k, d, c, so, do, ln, fl = f
    lo = k + d * U64(1 << 2) + c * U64(1 << 14) + so * U64(1 << 20) + (do % U64(4096)) * U64(1 << 52)
    hi = do // U64(4096) + ln * U64(1 << 20) + fl * U64(1 << 52)
    return lo, hi


def unpack_fields(lo, hi):
    """command.py:141-158."""
    lo = np.asarray(lo).astype(U64)
    hi = np.asarray(hi).astype(U64)
    if np.any(hi // U64(1 << 54)):
        raise CodecError("reserved bits")
    two32 = U64(1 << 32)
    return {
        "kind": (lo % U64(4)).astype(np.int64),
        "dst_rank": (lo // U64(4) % U64(4096)).astype(np.int64),
        "channel_id": (lo // U64(1 << 14) % U64(64)).astype(np.int64),
        "src_offset": (lo // U64(1 << 20) % two32).astype(np.int64),
        "dst_offset": ((lo // U64(1 << 52) + (hi % U64(1 << 20)) * U64(4096)) % two32).astype(np.int64),
        "length_or_value": (hi // U64(1 << 20) % two32).astype(np.int64),
        "flags": (hi // U64(1 << 52) % U64(4)).astype(np.int64),
    }


# --- immediate words (imm.py) ----------------------------------------------
SEQ_MOD, SEQ_WINDOW = 1 << 16, 1 << 15
HT_ROLE_HEAD, HT_DELTA_MASK = 0x80, 0x7F


def encode_ll(kind, counter_index, operand):  # imm.py:34-39
    if not 0 <= counter_index < 1024 or not 0 <= operand < (1 << 20):
        raise CodecError("ll field")
    return kind + 4 * counter_index + 4096 * operand


def decode_ll(imm):  # imm.py:42-44
    return imm % 4, (imm >> 2) % 1024, (imm >> 12) % (1 << 20)


def encode_ht(kind, channel_id, sequence, operand=0):  # imm.py:47-52
    if not 0 <= channel_id < 64 or not 0 <= operand < 256:
        raise CodecError("ht field")
    return kind + 4 * channel_id + 256 * (sequence % SEQ_MOD) + (operand << 24)


def decode_ht(imm):  # imm.py:55-57
    return imm % 4, (imm >> 2) % 64, (imm >> 8) % SEQ_MOD, (imm >> 24) % 256


def seq_delta(seq, expected):  # imm.py:60-66
    return (seq - expected) % SEQ_MOD


def ht_atomic_operand(advance_head, delta):  # imm.py:69-72
    if not 1 <= delta <= HT_DELTA_MASK:
        raise CodecError("delta")
    return (HT_ROLE_HEAD if advance_head else 0) + delta


def encode_ll_batch(kind, counter_index, operand):  # imm.py:75-78
    k, c, o = (np.asarray(a).astype(np.uint32) for a in (kind, counter_index, operand))
    return (k + c * np.uint32(4) + o * np.uint32(4096)).astype(np.int64)


def encode_ht_batch(kind, channel_id, sequence, operand):  # imm.py:81-91
    k, c, s, o = (np.asarray(a).astype(np.uint32) for a in (kind, channel_id, sequence, operand))
    return (k + c * np.uint32(4) + (s % np.uint32(SEQ_MOD)) * np.uint32(256) + o * np.uint32(1 << 24)).astype(np.int64)
