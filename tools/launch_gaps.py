"""Where the N=1 step's time goes between launches, on one clock.

Stamp kernels (epb_debug_stamp, %globaltimer) bracket every op in stream
order, with a device spin ahead so the host is never the bottleneck; the
kernels' own phase marks (EPB_TRACE=1) use the same clock.  Prints, per op,
the median of: stamp -> first mark of block 0 (launch latency), first -> last
mark (kernel span), last mark -> next stamp (tail), stamp -> stamp.
"""
import os
import statistics
import sys
from pathlib import Path

os.environ["EPB_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import ctypes as C
import numpy as np
import torch

import paper_2512_19849_b200 as epb
from paper_2512_19849_b200._lib import lib, raw_stream
from tests.helpers import bf16_random, make_routing, to_dev_bf16

H, E, K, T = 7168, 256, 8, 4096
g = np.random.default_rng(0)
idx, w = make_routing(g, T, E, K)
x = to_dev_bf16(bf16_random(g, (T, H)))
topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
buf = epb.Buffer(None, epb.nvl_bytes_hint(T, H, 1, K, 3))
st = torch.zeros(16, dtype=torch.int64, device="cuda")
spin = int(40e-6 * 1.9e9)


def stamp(i):
    lib.epb_debug_stamp(C.c_void_p(st.data_ptr() + 8 * i), C.c_void_p(raw_stream()))


def trace():
    tr = (C.c_int64 * 64)()
    lib.epb_trace(buf._rank.ctx, tr)
    return list(tr)


rows = {}
for it in range(40):
    torch.cuda._sleep(spin)
    stamp(0)
    torch.cuda._sleep(1)
    stamp(1)
    pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
    stamp(2)
    torch.cuda._sleep(spin)
    stamp(3)
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                         topk_idx=topk, topk_weights=wt)
    stamp(4)
    torch.cuda._sleep(spin)
    stamp(5)
    out, _, _ = buf.combine(rx, h, topk_weights=rtw)
    stamp(6)
    torch.cuda.synchronize()
    if it < 5:
        continue
    s = st.cpu().tolist()
    tr = trace()
    r = {"sleep(1) stamp->stamp": s[1] - s[0],
         "layout stamp->stamp": s[2] - s[1],
         "dispatch stamp->first mark": tr[0] - s[3], "dispatch first->all landed": tr[10] - tr[0],
         "dispatch last block mark->stamp": s[4] - max(tr[10], tr[12]), "dispatch stamp->stamp": s[4] - s[3],
         "combine stamp->entry": tr[15] - s[5], "combine entry->last reduce": tr[20] - tr[15],
         "combine last->stamp": s[6] - tr[20], "combine stamp->stamp": s[6] - s[5]}
    for k_, v in r.items():
        rows.setdefault(k_, []).append(v / 1e3)
for k_, v in rows.items():
    print(f"{k_:36s} {statistics.median(v):8.2f} us", flush=True)
buf.destroy()
