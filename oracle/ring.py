"""Oracle restatement of the SPSC batch ring over the int64 control array.

Layout kernels.py:23-31 (TAIL@0, HEAD@8, COMPLETED@16, FLAGS@24, slots from
32, two words per slot); batch semantics kernels.py:61-104: each pass moves
min(remaining, free-or-available) commands then publishes the owner's counter;
an empty/full observation counts one spin and the call returns a partial
count once spins exceed max_spin.  Single-threaded use only (the oracle is
checked on deterministic interleavings).
"""
from __future__ import annotations

import numpy as np

TAIL, HEAD, COMPLETED, FLAGS, SLOT0 = 0, 8, 16, 24, 32


def ctl_words(capacity: int) -> int:
    return SLOT0 + 2 * capacity


def _slot_index(counter: int, capacity: int) -> int:
    return SLOT0 + 2 * (counter % capacity)


def push_batch(ctl, cap, lo, hi, start, want, max_spin) -> int:
    tail = int(ctl[TAIL])
    done, spins = 0, 0
    while done < want:
        room = cap - (tail - int(ctl[HEAD]))
        if room <= 0:
            spins += 1
            if spins > max_spin:
                return done
            continue
        for _ in range(min(room, want - done)):
            s = _slot_index(tail, cap)
            ctl[s] = lo[start + done]
            ctl[s + 1] = hi[start + done]
            tail += 1
            done += 1
        ctl[TAIL] = tail
    return done


def pop_batch(ctl, cap, lo_out, hi_out, start, want, max_spin) -> int:
    head = int(ctl[HEAD])
    done, spins = 0, 0
    while done < want:
        ready = int(ctl[TAIL]) - head
        if ready <= 0:
            spins += 1
            if spins > max_spin:
                return done
            continue
        for _ in range(min(ready, want - done)):
            s = _slot_index(head, cap)
            lo_out[start + done] = ctl[s]
            hi_out[start + done] = ctl[s + 1]
            head += 1
            done += 1
        ctl[HEAD] = head
    return done


def new_ctl(capacity: int) -> np.ndarray:
    return np.zeros(ctl_words(capacity), np.int64)
