"""The proxies' all-peer barrier (Barrier TransferCmd, SPEC.md:274-282,
PAPER.md:313) on its host rendezvous alone: 'no participant returns before all
have entered', for every arrival order of 3 ranks, plus the
degenerate scopes.  CPU only: ranks are threads (ctypes releases the GIL)."""
import ctypes as C
import itertools
import os
import threading
import time
import uuid

import pytest

from paper_2512_19849_b200._lib import lib
from paper_2512_19849_b200.errors import raise_for


def _open(name, world, rank):
    b = C.c_void_p()
    raise_for(lib.epb_barrier_open(name.encode(), world, rank, C.byref(b)), lib.epb_last_error().decode())
    return b


def _name():
    return f"/epb_test_{os.getpid()}_{uuid.uuid4().hex[:12]}"


@pytest.mark.parametrize("order", list(itertools.permutations(range(3))))
def test_barrier_waits_for_last_arrival(order):
    name = _name()
    bars = [_open(name, 3, r) for r in range(3)]
    enter, leave = {}, {}

    def run(r):
        time.sleep(0.03 * order.index(r))  # arrival order
        enter[r] = time.monotonic()
        rc = lib.epb_barrier_wait(bars[r], 0, 10.0)
        leave[r] = time.monotonic()
        assert rc == 0

    for rep in range(2):  # consecutive epochs need no reset
        ts = [threading.Thread(target=run, args=(r,)) for r in range(3)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert min(leave.values()) >= max(enter.values()), (order, enter, leave)
    for r, b in enumerate(bars):
        lib.epb_barrier_close(b, int(r == 0))


def test_barrier_single_rank_and_same_rail():
    name = _name()
    b = _open(name, 1, 0)
    t0 = time.monotonic()
    assert lib.epb_barrier_wait(b, 0, 1.0) == 0  # 1 rank, AllPeers: immediate
    b2 = _open(_name(), 2, 0)
    assert lib.epb_barrier_wait(b2, 1, 1.0) == 0  # SameRail: no rail peers on one node
    assert time.monotonic() - t0 < 0.5
    lib.epb_barrier_close(b, 1)
    lib.epb_barrier_close(b2, 1)


def test_barrier_times_out_when_a_rank_is_absent():
    b = _open(_name(), 2, 0)
    rc = lib.epb_barrier_wait(b, 0, 0.2)
    assert rc != 0 and "absent" in lib.epb_last_error().decode()
    lib.epb_barrier_close(b, 1)
