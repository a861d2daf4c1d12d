"""Host-side (CPU) cost of each public API call on the N=1 DeepSeek-V3 step.

Prints mean wall-clock microseconds spent in Python/ctypes per call and the
top cProfile entries, to separate host overhead from device time.
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2512_19849_b200 as epb
from tests.helpers import bf16_random, make_routing, to_dev_bf16

T, H, E, K = 4096, 7168, 256, 8
g = np.random.default_rng(0)
idx, w = make_routing(g, T, E, K)
x = to_dev_bf16(bf16_random(g, (T, H)))
topk = torch.from_numpy(idx).cuda()
wt = torch.from_numpy(w).cuda()
buf = epb.Buffer(None, epb.nvl_bytes_hint(T, H, 1, K), epb.Buffer.get_low_latency_rdma_size_hint(128, H, 1, E, 8),
                 low_latency_mode=True)
acc = {"layout": 0.0, "dispatch": 0.0, "combine": 0.0, "ll_dispatch": 0.0, "ll_combine": 0.0}


def step(timed):
    t0 = time.perf_counter()
    per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(topk, E)
    t1 = time.perf_counter()
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank,
                                         num_tokens_per_expert=per_exp, topk_idx=topk, topk_weights=wt)
    t2 = time.perf_counter()
    out, ow, _ = buf.combine(rx, h, topk_weights=rtw)
    t3 = time.perf_counter()
    if timed:
        acc["layout"] += t1 - t0
        acc["dispatch"] += t2 - t1
        acc["combine"] += t3 - t2


xl = x[:128].contiguous()
tl = topk[:128].contiguous()
wl = wt[:128].contiguous()
y = torch.randn(E, 128, H, device="cuda").to(torch.bfloat16)


def ll(timed):
    t0 = time.perf_counter()
    recv, cnt, hd, _, _ = buf.low_latency_dispatch(xl, tl, 128, E)
    t1 = time.perf_counter()
    o, _, _ = buf.low_latency_combine(y, tl, wl, hd)
    t2 = time.perf_counter()
    if timed:
        acc["ll_dispatch"] += t1 - t0
        acc["ll_combine"] += t2 - t1


for _ in range(10):
    step(False)
    ll(False)
torch.cuda.synchronize()
N = 100
for _ in range(N):
    step(True)
torch.cuda.synchronize()
for _ in range(N):
    torch.cuda._sleep(2_000_000)  # keep the GPU busy so host calls never wait on it
    ll(True)
torch.cuda.synchronize()
print({k: round(v / N * 1e6, 1) for k, v in acc.items()}, "us of host time per call")
pr = cProfile.Profile()
pr.enable()
for _ in range(30):
    step(False)
for _ in range(30):
    ll(False)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
