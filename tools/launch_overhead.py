"""Per-op device time of the N=1 step, measured three ways:

* `events`: CUDA events around each op with a device spin queued ahead (the
  bench's profiled pass), i.e. launch-to-completion on the GPU;
* `span`  : globaltimer marks inside the kernels (EPB_TRACE=1): first mark of
  block 0 to the last block's last mark;
* `graph` : the same op replayed from a CUDA graph (dispatch with a cached
  handle, which has no host wait), back to back.

    EPB_COOP=0|1 python tools/launch_overhead.py
"""
import os
import statistics
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
buf = epb.Buffer(None, epb.nvl_bytes_hint(T, H, 1, K, 3))
spin = int(30e-6 * 1.9e9)
prof = []
for i in range(60):
    on = i >= 10
    if on:
        epb.buffer.X.set_profiling(True)
    torch.cuda._sleep(spin)
    pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
    torch.cuda._sleep(spin)
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                         topk_idx=topk, topk_weights=wt)
    torch.cuda._sleep(spin)
    out, _, _ = buf.combine(rx, h, topk_weights=rtw)
    if on:
        epb.buffer.X.set_profiling(False)
        prof.extend(epb.buffer.X.collect_profile())
torch.cuda.synchronize()
per = {}
for name, ms in prof:
    per.setdefault(name, []).append(ms * 1e3)
print(f"EPB_COOP={os.environ.get('EPB_COOP', '1')} events (spin ahead), median us:",
      {k: round(statistics.median(v), 2) for k, v in per.items()}, flush=True)

# back-to-back eager (no spin): what the step sees
for name, fn in (("layout", lambda: buf.get_dispatch_layout(topk, E)),
                 ("combine", lambda: buf.combine(rx, h, topk_weights=rtw)),
                 ("dispatch_cached", lambda: buf.dispatch(x, handle=h, topk_idx=None, topk_weights=None))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(spin * 4)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"  {name}: back-to-back {e0.elapsed_time(e1) / 50 * 1e3:.2f} us/op", flush=True)
buf.destroy()
