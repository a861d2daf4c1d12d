"""The GPU->CPU command channel beyond the data paths (PAPER.md:302-315,
SPEC.md:264-282): Drain(Idx) pushed by a kernel and completed by the CPU proxy
once the copies of commands <= Idx have landed; proxy error reporting; the
phase trace of the LL proxy transport (host events on the GPU clock)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    assert _t.cuda.is_available()
    return _t


def _buf(nvl, **kw):
    from paper_2512_19849_b200 import Buffer
    return Buffer(None, nvl, 1 << 20, low_latency_mode=True, fifo_channels=4, proxy_threads=2, ll_transport="proxy",
                  **kw)


@pytest.mark.parametrize("upto", [4, -1])
def test_drain_idx(torch, upto):
    """A kernel pushes 10 WRITEs of 32 MB on one channel, then Drain(upto-th WRITE)
    and spins on check_completion: when the drain completes, every block <= upto
    has landed (all of them for a full drain)."""
    from paper_2512_19849_b200._lib import check, lib, raw_stream
    n, nbytes = 10, 32 << 20
    buf = _buf(2 * n * nbytes + (4 << 20))
    arena = lib.epb_arena_offset()
    region = buf.get_local_buffer_tensor(torch.uint8)
    src = region[arena: arena + n * nbytes].view(n, nbytes)
    dst = region[arena + n * nbytes: arena + 2 * n * nbytes].view(n, nbytes)
    for i in range(n):
        src[i].fill_(i + 1)
    dst.zero_()
    res = torch.zeros(n + 1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    check(lib.epb_debug_drain_test(buf._rank.ctx, 1, 0, n, 0, n * nbytes, nbytes, upto, res.data_ptr(), raw_stream()))
    torch.cuda.synchronize()
    buf._g.check_device_error()
    r = res.cpu().numpy()
    last = n - 1 if upto < 0 else upto
    assert (r[: last + 1] == 1).all(), r
    print(f"drain(upto={upto}): landed {r[:n].tolist()}, push->complete {r[n] / 1e3:.1f} us")
    # every copy is done eventually (stream order), and the data is right
    torch.cuda.synchronize()
    check(lib.epb_proxy_drain(buf._rank.ctx, 1, -1, raw_stream()))
    torch.cuda.synchronize()
    for i in range(n):
        assert int(dst[i, 0]) == i + 1 and int(dst[i, -1]) == i + 1
    buf.destroy()


def test_proxy_reports_fault(torch):
    """An out-of-bounds WRITE is rejected by the proxy with FaultError (errors.py:20-27)
    instead of being issued; the drain behind it still completes."""
    from paper_2512_19849_b200._lib import check, lib, raw_stream
    from paper_2512_19849_b200.errors import FaultError
    buf = _buf(1 << 20)
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    check(lib.epb_debug_drain_test(buf._rank.ctx, 0, 0, 1, 0, 1 << 30, 1 << 20, -1, res.data_ptr(), raw_stream()))
    torch.cuda.synchronize()
    with pytest.raises(FaultError):
        buf._g.check_device_error()
    buf.destroy()


def test_ll_proxy_trace_and_clock(torch):
    """EPB_TRACE=1: the LL proxy pair records its group pushes on the GPU and the
    proxy's tail/copy/signal events on the host; after clock calibration the host
    events fall between the kernel's first push and the receiver's wake-up."""
    import os
    from paper_2512_19849_b200 import LocalGroup
    from paper_2512_19849_b200._lib import lib
    from tests.helpers import bf16_random, make_routing, to_dev_bf16
    os.environ["EPB_TRACE"] = "1"
    try:
        R, T, H, E, k = 2, 64, 2048, 16, 4
        from paper_2512_19849_b200 import Buffer
        ll_bytes = Buffer.get_low_latency_rdma_size_hint(T, H, R, E, num_topk=k)
        grp = LocalGroup(R, 1 << 20, ll_bytes, fifo_channels=8, proxy_threads=2, ll_transport="proxy")
    finally:
        del os.environ["EPB_TRACE"]
    off, err = C.c_int64(), C.c_int64()
    assert lib.epb_clock_calibrate(C.byref(off), C.byref(err)) == 0
    assert err.value < 20_000, err.value  # the host bracket around a beacon read
    g = np.random.default_rng(0)
    xs = [to_dev_bf16(bf16_random(g, (T, H))) for _ in range(R)]
    idx = [torch.from_numpy(make_routing(g, T, E, k)[0]).cuda() for _ in range(R)]
    for _ in range(3):
        res, _ = grp.low_latency_dispatch(xs, idx, T, E, use_fp8=True)
    torch.cuda.synchronize()
    grp.check_device_error()
    marks = (C.c_int64 * 64)()
    assert lib.epb_trace(grp.ranks[0].ctx, marks) == 0
    for rk in grp.ranks:
        lib.epb_proxy_stop(rk.ctx)
    n = lib.epb_proxy_trace(grp.ranks[0].ctx, None, 0)
    ev = (C.c_int64 * (4 * n))()
    lib.epb_proxy_trace(grp.ranks[0].ctx, ev, n)
    evs = np.frombuffer(ev, np.int64).reshape(n, 4)
    kinds = set(evs[:, 1].tolist())
    assert {1, 2, 3} <= kinds, kinds  # tail seen, copy issued, signal issued
    pushes = [marks[40 + gi] for gi in range(4) if marks[40 + gi]]
    assert pushes
    wake = marks[28]
    host_on_gpu = evs[:, 0] + off.value
    last_call = host_on_gpu[host_on_gpu >= min(pushes) - 50_000]
    assert len(last_call), "no proxy event near the last call's pushes"
    assert (last_call[last_call <= wake + 50_000]).size > 0
    for rk in grp.ranks:
        rk.proxy_running = False
    grp.destroy()
