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
NAMES = {0: "notify start", 1: "count", 2: "scan", 3: "post msgs", 4: "wait peers", 5: "prefix+per-expert",
         6: "publish", 8: "dispatch start", 9: "copies done", 10: "all arrived", 16: "combine start",
         17: "push done", 18: "barrier", 19: "reduce done", 24: "ll_disp start", 25: "bitmap", 26: "items done",
         27: "ticket", 28: "recv wait", 33: "ll_comb items", 34: "ll_comb wait"}


def show(label):
    tr = (C.c_int64 * 64)()
    lib.epb_trace(buf._rank.ctx, tr)
    ts = {i: tr[i] for i in range(64) if tr[i]}
    print(label)
    groups = [(0, 6), (8, 10), (16, 19), (24, 28), (32, 35)]
    for a, b in groups:
        keys = [k for k in sorted(ts) if a <= k <= b]
        if not keys:
            continue
        t0 = ts[keys[0]]
        print("   " + "  ".join(f"{NAMES.get(k, k)}=+{(ts[k] - t0) / 1e3:.2f}us" for k in keys))


for i in range(6):
    pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                         topk_idx=topk, topk_weights=wt)
    out, _, _ = buf.combine(rx, h, topk_weights=rtw)
    torch.cuda.synchronize()
show("normal (EP=1, 4096 tokens)")
for i in range(6):
    recv, cnt, hd, _, _ = buf.low_latency_dispatch(x[:128].contiguous(), topk[:128].contiguous(), 128, E)
    o, _, _ = buf.low_latency_combine(y, topk[:128].contiguous(), wt[:128].contiguous(), hd)
    torch.cuda.synchronize()
show("low latency (EP=1, 128 tokens)")
buf.destroy()
