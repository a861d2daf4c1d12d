"""Per-phase device timestamps of the N=1 kernels (EPB_TRACE=1 must be set).

Runs a few normal and LL steps and prints the intervals between the phase
marks recorded by block 0 / thread 0 (see trace_mark() calls in csrc/).
"""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["EPB_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2512_19849_b200 as epb
from paper_2512_19849_b200._lib import lib
from tests.helpers import bf16_random, make_routing, to_dev_bf16

H, E, K = 7168, 256, 8
g = np.random.default_rng(0)
T = 4096
idx, w = make_routing(g, T, E, K)
x = to_dev_bf16(bf16_random(g, (T, H)))
topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
buf = epb.Buffer(None, epb.nvl_bytes_hint(T, H, 1, K), epb.Buffer.get_low_latency_rdma_size_hint(128, H, 1, E, K),
                 low_latency_mode=True)
y = torch.randn(E, 128, H, device="cuda").to(torch.bfloat16)
NAMES = {2: "gather start", 0: "dispatch start", 1: "all channels counted", 3: "msgs posted", 4: "peers' msgs",
         5: "plan published", 6: "host counts", 7: "block0 copy start", 9: "block0 copies done", 10: "all rows landed",
         15: "combine entry", 16: "combine start", 17: "push done", 18: "barrier", 19: "reduce done", 24: "ll_disp start", 25: "bitmap",
         26: "items done", 27: "ticket", 28: "recv wait", 29: "ll_disp last block done", 32: "ll_comb start", 33: "ll_comb items", 34: "ll_comb wait", 35: "ll_comb last block done", 11: "last block copy start", 12: "last block copies done", 20: "last block reduce done", 21: "last block reduce start"}


def snap():
    tr = (C.c_int64 * 64)()
    lib.epb_trace(buf._rank.ctx, tr)
    return {i: tr[i] for i in range(64) if tr[i]}


def show(label, snaps):
    """Median over calls of each mark's offset from the first mark of its group."""
    import statistics
    print(label, flush=True)
    for a, b in [(0, 12), (15, 21), (24, 29), (32, 35)]:
        offs = {}
        for ts in snaps:
            keys = [k for k in sorted(ts) if a <= k <= b]
            if not keys:
                continue
            for k in keys:
                offs.setdefault(k, []).append((ts[k] - ts[keys[0]]) / 1e3)
        if offs:
            print("   " + "  ".join(f"{NAMES.get(k, k)}=+{statistics.median(v):.2f}us"
                                    for k, v in sorted(offs.items(), key=lambda kv: statistics.median(kv[1]))),
                  flush=True)


snaps = []
for i in range(35):
    pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                         topk_idx=topk, topk_weights=wt)
    out, _, _ = buf.combine(rx, h, topk_weights=rtw)
    torch.cuda.synchronize()
    if i >= 5:
        snaps.append(snap())
show("normal (EP=1, 4096 tokens), median of 30 calls", snaps)
snaps = []
for i in range(35):
    recv, cnt, hd, _, _ = buf.low_latency_dispatch(x[:128].contiguous(), topk[:128].contiguous(), 128, E)
    o, _, _ = buf.low_latency_combine(y, topk[:128].contiguous(), wt[:128].contiguous(), hd)
    torch.cuda.synchronize()
    if i >= 5:
        snaps.append({k: v for k, v in snap().items() if k >= 24})
show("low latency (EP=1, 128 tokens), median of 30 calls", snaps)
buf.destroy()
