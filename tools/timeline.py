"""GPU timeline of the N=1 normal step via torch.profiler (CUPTI): kernel
durations and the idle gaps between consecutive kernels, to separate device
time from host-side launch gaps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2512_19849_b200 as epb
from tests.helpers import bf16_random, make_routing, to_dev_bf16

T, H, E, K = 4096, 7168, 256, 8
g = np.random.default_rng(0)
idx, w = make_routing(g, T, E, K)
x = to_dev_bf16(bf16_random(g, (T, H)))
topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
buf = epb.Buffer(None, epb.nvl_bytes_hint(T, H, 1, K))


def step():
    pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                         topk_idx=topk, topk_weights=wt)
    out, _, _ = buf.combine(rx, h, topk_weights=rtw)


for _ in range(10):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(10):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
prev_end = None
rows = []
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    gap = (s - prev_end) if prev_end is not None else 0
    rows.append((e.name[:40], t - s, gap))
    prev_end = t
tot = {}
for n, d, gp in rows:
    a = tot.setdefault(n, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d
    a[2] += gp
span = evs[-1].time_range.end - evs[0].time_range.start
print(f"span of 10 steps: {span:.1f} us -> {span / 10:.1f} us/step")
for n, (c, d, gp) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:42s} n={c:3d} busy={d / c:8.2f} us  gap-before={gp / c:7.2f} us")
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
