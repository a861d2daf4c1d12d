"""Chunked-ring transport (ht_transport="ring") at N=1, DS-V3 shape: dispatch
and combine device time per (lanes, ring slots) setting, arena bytes beside."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2512_19849_b200 as epb
from tests.helpers import bf16_random, make_routing, to_dev_bf16

H, E, K, T = 7168, 256, 8, 4096
g = np.random.default_rng(0)
idx, w = make_routing(g, T, E, K)
x = to_dev_bf16(bf16_random(g, (T, H)))
topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
for lanes, slots in [(16, 256), (32, 128), (48, 128), (74, 64), (74, 128)]:
    nvl = epb.ring_nvl_bytes(H, 1, K, lanes, slots)
    buf = epb.Buffer(None, nvl, ht_transport="ring", ring_lanes=lanes)
    ts = []
    for it in range(12):
        pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda._sleep(40000)
        e[0].record()
        rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                             topk_idx=topk, topk_weights=wt)
        e[1].record()
        torch.cuda._sleep(40000)
        e[2].record()
        buf.combine(rx, h, topk_weights=rtw)
        e[3].record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append((e[0].elapsed_time(e[1]) * 1e3, e[2].elapsed_time(e[3]) * 1e3))
    d = float(np.median([t[0] for t in ts]))
    c = float(np.median([t[1] for t in ts]))
    print(f"lanes {lanes:3d} slots {slots:4d} arena {nvl / 1e6:7.1f} MB: dispatch {d:7.1f} us  combine {c:7.1f} us",
          flush=True)
    buf.destroy()
