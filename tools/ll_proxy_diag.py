"""Diagnose the LL proxy transport on one GPU: per-call device time, proxy
counters and FIFO state; with EPB_TRACE the proxy's API-call costs.
    python tools/ll_proxy_diag.py [--trace] [--calls 10] [--channels 16] [--threads 4] [--ranks 1]"""
import argparse
import ctypes as C
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--trace", action="store_true")
ap.add_argument("--calls", type=int, default=10)
ap.add_argument("--channels", type=int, default=16)
ap.add_argument("--threads", type=int, default=4)
ap.add_argument("--ranks", type=int, default=1)
ap.add_argument("--buffer", action="store_true", help="one-rank Buffer instead of LocalGroup")
ap.add_argument("--calibrate", action="store_true", help="run epb_clock_calibrate first")
ap.add_argument("--sync-trace", action="store_true", help="read the kernel trace words after every call")
args = ap.parse_args()
if args.trace:
    os.environ["EPB_TRACE"] = "1"
os.environ.setdefault("EPB_TIMEOUT_S", "3")
import numpy as np
import torch

import paper_2512_19849_b200 as epb
from paper_2512_19849_b200._lib import lib
from tests.helpers import bf16_random, make_routing

T, H, E, k, R = 128, 7168, 256, 8, args.ranks
ll = epb.Buffer.get_low_latency_rdma_size_hint(T, H, R, E, num_topk=k)
if args.buffer:
    b = epb.Buffer(None, 1 << 20, ll, low_latency_mode=True, fifo_channels=args.channels, proxy_threads=args.threads,
                   ll_transport="proxy")

    class _G:  # LocalGroup-like view of the one-rank Buffer
        ranks = [b._rank]

        def low_latency_dispatch(self, xs_, ti_, T_, E_, use_fp8=True):
            r = b.low_latency_dispatch(xs_[0], ti_[0], T_, E_, use_fp8=use_fp8)
            return [(r[0], r[1], r[2])], None

        def low_latency_combine(self, ys_, ti_, tw_, hs_):
            return [b.low_latency_combine(ys_[0], ti_[0], tw_[0], hs_[0])[0]], None

        def check_device_error(self):
            b._g.check_device_error()

        def destroy(self):
            b.destroy()
    grp = _G()
else:
    grp = epb.LocalGroup(R, 1 << 20, ll, fifo_channels=args.channels, proxy_threads=args.threads,
                         ll_transport="proxy")
if args.calibrate:
    off, err = C.c_int64(), C.c_int64()
    print("calibrate rc", lib.epb_clock_calibrate(C.byref(off), C.byref(err)), off.value, err.value, flush=True)
g = np.random.default_rng(0)
xs = [torch.from_numpy(bf16_random(g, (T, H)).view(np.int16)).view(torch.bfloat16).cuda() for _ in range(R)]
idx = [make_routing(g, T, E, k) for _ in range(R)]
ti = [torch.from_numpy(i).cuda() for i, _ in idx]
tw = [torch.from_numpy(w).cuda() for _, w in idx]
y = [torch.randn(E // R, R * T, H, device="cuda").to(torch.bfloat16) for _ in range(R)]


def state(tag):
    rk = grp.ranks[0]
    st = (C.c_int64 * 3)()
    lib.epb_proxy_stats(rk.ctx, st)
    ctl = []
    for ch in range(args.channels):
        q, cap = C.POINTER(C.c_int64)(), C.c_int64()
        lib.epb_fifo_ctl(rk.ctx, ch, C.byref(q), C.byref(cap))
        ctl.append((q[0], q[8], q[16]))
    meta = torch.as_tensor(epb.buffer._SlotMemory(rk.base, 192 + 64 * 8 * 8), device="cuda").cpu().numpy()
    sig = meta[192:].view(np.uint64).reshape(64, 8)
    print(f"[{tag}] served/copies/writes {list(st)}; ctl(tail,head,completed) {ctl}", flush=True)
    print(f"   proxy_sig disp {sig[:args.threads, :R].tolist()} comb {sig[32:32 + args.threads, :R].tolist()}", flush=True)


dts = []
for i in range(args.calls):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    res, _ = grp.low_latency_dispatch(xs, ti, T, E, use_fp8=True)
    e1.record()
    grp.low_latency_combine(y, ti, tw, [r[2] for r in res])
    e2.record()
    torch.cuda.synchronize()
    dts.append((e0.elapsed_time(e1) * 1e3, e1.elapsed_time(e2) * 1e3))
    if args.sync_trace:
        m = (C.c_int64 * 64)()
        lib.epb_trace(grp.ranks[0].ctx, m)
    try:
        grp.check_device_error()
    except Exception as exc:  # noqa: BLE001
        print(f"call {i}: {exc}", flush=True)
        state(f"after call {i}")
        break
print("dispatch / combine us per call:", [(round(a, 1), round(b, 1)) for a, b in dts], flush=True)
state("end")
if args.trace:
    for rk in grp.ranks:
        lib.epb_proxy_stop(rk.ctx)
        rk.proxy_running = False
    n = lib.epb_proxy_trace(grp.ranks[0].ctx, None, 0)
    ev = (C.c_int64 * (4 * max(1, n)))()
    lib.epb_proxy_trace(grp.ranks[0].ctx, ev, n)
    evs = np.frombuffer(ev, np.int64)[: 4 * n].reshape(n, 4)
    cost = {6: [], 7: [], 8: []}
    after = {6: 2, 7: 3, 8: 9}
    for j in range(n - 1):
        kd = int(evs[j, 1])
        if kd in cost:
            nxt = [m for m in range(j + 1, min(n, j + 8)) if evs[m, 1] == after[kd]]
            if nxt:
                cost[kd].append((evs[nxt[0], 0] - evs[j, 0]) / 1e3)
    for kd, name in ((6, "cudaMemcpyAsync"), (7, "cuStreamWriteValue64"), (8, "cudaEventRecord")):
        if cost[kd]:
            print(f"{name:22s} n={len(cost[kd])} median {statistics.median(cost[kd]):.2f} us max {max(cost[kd]):.2f} us")
    print("events by kind:", {int(kd): int((evs[:, 1] == kd).sum()) for kd in np.unique(evs[:, 1])})
grp.destroy()
