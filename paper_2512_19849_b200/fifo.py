"""FifoChannel: the bounded lock-free SPSC command channel.

Backed by an int64 control array in the reference layout (kernels.py:23-31).
The array is either a private numpy array (CPU producer and consumer) or the
pinned, device-mapped control array of one of a Buffer's GPU->CPU FIFOs (GPU
producer, CPU proxy consumer).  All operations run in the C ABI with
release/acquire ordering.

Command indices are the 0-based push order.  ``mark_completed(upto)`` and
``check_completion(idx)`` follow SPEC.md:80-98 (completed_upto starts below 0,
so a fresh push is not complete).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import command
from ._lib import lib, nptr
from .errors import ChannelShutdown, ProtocolViolation

CTL_TAIL, CTL_HEAD, CTL_COMPLETED, CTL_FLAGS, CTL_SLOT0 = 0, 8, 16, 24, 32


class FifoChannel:
    def __init__(self, capacity: int = 64, ctl: Optional[np.ndarray] = None, spin: int = 1 << 20):
        if capacity <= 0 or capacity & (capacity - 1):
            raise ProtocolViolation("capacity must be a power of two (SPEC.md:108)")
        self.capacity = capacity
        self.ctl = ctl if ctl is not None else np.zeros(CTL_SLOT0 + 2 * capacity, np.int64)
        self._p = nptr(self.ctl, C.c_int64)
        self._spin = spin
        self._one_lo = np.zeros(1, np.int64)
        self._one_hi = np.zeros(1, np.int64)

    # producer side ---------------------------------------------------------
    def push(self, cmd: command.TransferCmd, block: bool = True) -> int:
        lo, hi = command.pack(cmd)
        self._one_lo[0] = np.array([lo], np.uint64).view(np.int64)[0]
        self._one_hi[0] = np.array([hi], np.uint64).view(np.int64)[0]
        while True:
            idx = int(self.ctl[CTL_TAIL])
            r = lib.epb_ring_push_batch(self._p, self.capacity, nptr(self._one_lo, C.c_int64),
                                        nptr(self._one_hi, C.c_int64), 0, 1, self._spin)
            if r < 0:
                raise ChannelShutdown("channel shut down")
            if r == 1:
                return idx
            if not block:
                raise ProtocolViolation("channel full")

    def shutdown(self) -> None:
        lib.epb_ring_shutdown(self._p)

    # consumer side -----------------------------------------------------------
    def poll(self) -> Optional[command.TransferCmd]:
        lo, hi = C.c_int64(), C.c_int64()
        if not lib.epb_ring_poll(self._p, self.capacity, C.byref(lo), C.byref(hi)):
            return None
        return command.unpack(lo.value & (2**64 - 1), hi.value & (2**64 - 1))

    def pop(self) -> command.TransferCmd:
        lo = np.zeros(1, np.int64)
        hi = np.zeros(1, np.int64)
        if lib.epb_ring_pop_batch(self._p, self.capacity, nptr(lo, C.c_int64), nptr(hi, C.c_int64), 0, 1, 0) != 1:
            raise ProtocolViolation("pop on empty channel")
        return command.unpack(int(lo.view(np.uint64)[0]), int(hi.view(np.uint64)[0]))

    def mark_completed(self, upto: int) -> None:
        if lib.epb_ring_mark_completed(self._p, int(upto) + 1) != 0:
            raise ProtocolViolation(f"mark_completed({upto}) beyond head {int(self.ctl[CTL_HEAD])}")

    def check_completion(self, idx: int) -> bool:
        return bool(lib.epb_ring_check_completion(self._p, int(idx)))

    @property
    def head(self) -> int:
        return int(self.ctl[CTL_HEAD])

    @property
    def tail(self) -> int:
        return int(self.ctl[CTL_TAIL])

    @property
    def completed_upto(self) -> int:
        return int(self.ctl[CTL_COMPLETED]) - 1
