"""Host (CPU) cost per public API call with negligible device work (64 tokens),
so that the wall time per call is the Python + C++ + launch overhead.  The
dispatch figure also contains one device round trip (the receive counts)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2512_19849_b200 as epb
from tests.helpers import bf16_random, make_routing, to_dev_bf16

T, H, E, K = 64, 7168, 256, 8
g = np.random.default_rng(0)
idx, w = make_routing(g, T, E, K)
x = to_dev_bf16(bf16_random(g, (T, H)))
topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
buf = epb.Buffer(None, epb.nvl_bytes_hint(4096, H, 1, K))
pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                     topk_idx=topk, topk_weights=wt)
N = 2000


def timed(name, fn):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:28s} {(t1 - t0) / N * 1e6:7.2f} us/call (host)", flush=True)


timed("empty torch op (x.view)", lambda: x.view(-1))
timed("get_dispatch_layout", lambda: buf.get_dispatch_layout(topk, E))
timed("dispatch", lambda: buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                       topk_idx=topk, topk_weights=wt))
from paper_2512_19849_b200 import _epb_ext as X  # noqa: E402
X.host_timers()
timed("dispatch (again)", lambda: buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir,
                                               num_tokens_per_expert=pe, topk_idx=topk, topk_weights=wt))
print("   dispatch phases:", {k: round(v, 2) if isinstance(v, float) else v for k, v in X.host_timers().items()})
timed("combine", lambda: buf.combine(rx, h, topk_weights=rtw))


def step():
    pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                         topk_idx=topk, topk_weights=wt)
    buf.combine(rx, h, topk_weights=rtw)


timed("step (layout+dispatch+combine)", step)
buf.destroy()
