"""Phase trace of the low-latency pair through the GPU->CPU FIFO + CPU proxy.

    python tools/trace_ll_proxy.py [--calls 30]                   # 1 GPU
    torchrun --nproc-per-node N tools/trace_ll_proxy.py ...         # N GPUs

With EPB_TRACE=1 the LL kernels record %globaltimer marks (kernel start, each
command group's push, receiver wake-up, end) and the proxy threads record host
events (tail seen, copy issued, value write issued).  The host clock is put on
the GPU clock with epb_clock_calibrate.  Per call, for dispatch and combine:

    start -> first push -> host sees first tail -> first copy issued
          -> last signal issued -> receiver wakes -> done        (us, median over calls)
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ["EPB_TRACE"] = "1"
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=30)
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--fifo-channels", type=int, default=16)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    group = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        group = dist.group.WORLD
    import paper_2512_19849_b200 as epb
    from paper_2512_19849_b200._lib import lib
    from tests.helpers import bf16_random, make_routing
    T, H, E, k = args.tokens, 7168, 256, 8
    buf = epb.Buffer(group, 1 << 20, epb.Buffer.get_low_latency_rdma_size_hint(T, H, world, E, num_topk=k),
                     low_latency_mode=True, fifo_channels=args.fifo_channels, ll_transport="proxy")
    g = np.random.default_rng(rank)
    x = torch.from_numpy(bf16_random(g, (T, H)).view(np.int16)).view(torch.bfloat16).cuda()
    idx, w = make_routing(g, T, E, k)
    ti, tw = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
    y = torch.randn(E // world, world * T, H, device="cuda").to(torch.bfloat16)
    off, err = C.c_int64(), C.c_int64()
    lib.epb_clock_calibrate(C.byref(off), C.byref(err))
    calls = []
    for i in range(args.calls + 5):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        _, _, handle, _, _ = buf.low_latency_dispatch(x, ti, T, E, use_fp8=True)
        buf.low_latency_combine(y, ti, tw, handle)
        torch.cuda.synchronize()
        m = (C.c_int64 * 64)()
        lib.epb_trace(buf._rank.ctx, m)
        try:
            buf._g.check_device_error()
        except Exception as exc:  # noqa: BLE001  (a timed-out warm-up call: report, keep going)
            st = (C.c_int64 * 16)()
            lib.epb_debug_ll_state(buf._rank.ctx, st)
            ps = (C.c_int64 * 3)()
            lib.epb_proxy_stats(buf._rank.ctx, ps)
            ctl = []
            for ch in range(args.fifo_channels):
                q, cap = C.POINTER(C.c_int64)(), C.c_int64()
                lib.epb_fifo_ctl(buf._rank.ctx, ch, C.byref(q), C.byref(cap))
                ctl.append((q[0], q[8], q[16]))
            meta = torch.as_tensor(epb.buffer._SlotMemory(buf._rank.base, 192 + 64 * 64), device="cuda").cpu().numpy()
            sig = meta[192:].view(np.uint64).reshape(64, 8)
            print(f"call {i} rank {rank}: {exc}; llp_self/pcnt/epoch/grp {list(st)} proxy {list(ps)} ctl {ctl} "
                  f"sig disp {sig[:4, :world].tolist()} comb {sig[32:36, :world].tolist()}", file=sys.stderr, flush=True)
            continue
        if i >= 5:
            calls.append(list(m))
    lib.epb_proxy_stop(buf._rank.ctx)
    buf._rank.proxy_running = False
    n = lib.epb_proxy_trace(buf._rank.ctx, None, 0)
    ev = (C.c_int64 * (4 * max(1, n)))()
    lib.epb_proxy_trace(buf._rank.ctx, ev, n)
    evs = np.frombuffer(ev, np.int64)[: 4 * n].reshape(n, 4).copy()
    host_ev = evs[:, 1] < 10  # kinds >= 10: device stamps (already on the GPU clock)
    evs[host_ev, 0] += off.value  # host events on the GPU clock
    evs = evs[np.argsort(evs[:, 0], kind="stable")]
    G = args.fifo_channels // 2

    def phases(m, start, stage, push0, wake, done, chan_lo):
        pushes = [m[push0 + j] for j in range(min(G, 12)) if m[push0 + j] >= m[start]]
        if not pushes:
            return None
        p0, p1 = min(pushes), max(pushes)
        win = evs[(evs[:, 0] >= p0 - 2000) & (evs[:, 0] <= m[wake] + 2000)]
        tail = win[(win[:, 1] == 1) & (win[:, 2] >= chan_lo) & (win[:, 2] < chan_lo + G)]
        cp = win[win[:, 1] == 2]
        sig = win[win[:, 1] == 3]
        t0 = m[start]

        def rel(v):
            return round((v - t0) / 1e3, 2)
        return {"prologue": rel(m[stage - 1]) if start == 24 else None, "staged": rel(m[stage]),
                "first_push": rel(p0), "last_push": rel(p1),
                "host_sees_tail": rel(tail[0, 0]) if len(tail) else None,
                "first_copy_issued": rel(cp[0, 0]) if len(cp) else None,
                "last_signal_issued": rel(sig[-1, 0]) if len(sig) else None,
                "copy_kernel_start": rel(win[win[:, 1] == 10][0, 0]) if (win[:, 1] == 10).any() else None,
                "copy_kernel_last_block_start": rel(win[win[:, 1] == 12][-1, 0]) if (win[:, 1] == 12).any() else None,
                "copy_kernel_copies_done": rel(win[win[:, 1] == 13][-1, 0]) if (win[:, 1] == 13).any() else None,
                "copy_kernel_last_signal": rel(win[win[:, 1] == 11][-1, 0]) if (win[:, 1] == 11).any() else None,
                "receiver_wakes": rel(m[wake]), "done": rel(m[done])}

    if calls and len(evs):  # alignment sanity (stderr): the last call's marks vs the nearest host events
        m = calls[-1]
        near = evs[np.argsort(np.abs(evs[:, 0] - m[24]))[:6]]
        print(f"last call marks start {m[24]} staged {m[26]} wake {m[28]}; nearest host events "
              f"{[(int(e[0] - m[24]), int(e[1])) for e in near]}", file=sys.stderr, flush=True)
    out = {"rank": rank, "world": world, "tokens": T, "fifo_channels": args.fifo_channels,
           "groups_per_rank": int(os.environ.get("EPB_LL_GROUPS_PER_RANK", "1")),
           "clock_offset_ns": off.value, "clock_error_ns": err.value, "calls": len(calls)}
    for name, spec in (("dispatch", (24, 26, 40, 28, 29, 0)), ("combine", (32, 33, 52, 34, 35, G))):
        rows = [p for p in (phases(m, *spec) for m in calls) if p]
        med = {}
        for key in rows[0] if rows else []:
            vals = [r[key] for r in rows if r.get(key) is not None]
            med[key] = round(statistics.median(vals), 2) if vals else None
        out[name] = med
    # kernel-internal marks (us after the phase's kernel start, block 0 unless "last")
    for name, t0, keys in (("dispatch_marks", 24, {"last_block_start": 39, "bitmap": 30, "counts": 62, "rs_zeroed": 63, "routing_scan": 31,
                                                   "prologue": 25, "last_block_staged": 36, "block0_done": 26}),
                           ("combine_marks", 32, {"last_block_staged": 37, "push_entry": 60, "push_fenced": 61,
                                                  "block0_done": 33})):
        out[name] = {key: round(statistics.median([(m[i] - m[t0]) / 1e3 for m in calls]), 2) if calls else None
                     for key, i in keys.items()}
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(f"{args.out}.r{rank}.json", "w") as f:
            f.write(line + "\n")
    buf.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
