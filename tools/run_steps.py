"""Run a few N=1 steps of one path (for ncu / compute-sanitizer captures).

    python tools/run_steps.py normal|ll [steps]

`ll` uses the direct NVLink transport only (the proxy transport cannot make
progress under a kernel-serialising profiler).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2512_19849_b200 as epb
from tests.helpers import bf16_random, make_routing, to_dev_bf16

mode = sys.argv[1] if len(sys.argv) > 1 else "normal"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
H, E, K = 7168, 256, 8
g = np.random.default_rng(0)
if mode == "normal":
    T = 4096
    idx, w = make_routing(g, T, E, K)
    x = to_dev_bf16(bf16_random(g, (T, H)))
    topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
    buf = epb.Buffer(None, epb.nvl_bytes_hint(T, H, 1, K))
    for _ in range(steps):
        pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
        rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir,
                                             num_tokens_per_expert=pe, topk_idx=topk, topk_weights=wt)
        out, _, _ = buf.combine(rx, h, topk_weights=rtw)
else:
    T = 128
    idx, w = make_routing(g, T, E, K)
    x = to_dev_bf16(bf16_random(g, (T, H)))
    topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
    buf = epb.Buffer(None, 1 << 20, epb.Buffer.get_low_latency_rdma_size_hint(T, H, 1, E, num_topk=K),
                     low_latency_mode=True)
    y = torch.randn(E, T, H, device="cuda").to(torch.bfloat16)
    for _ in range(steps):
        recv, cnt, hd, _, _ = buf.low_latency_dispatch(x, topk, T, E)
        out, _, _ = buf.low_latency_combine(y, topk, wt, hd)
torch.cuda.synchronize()
buf.destroy()
print("ok")
