"""Per-phase device timestamps at EP=N (run under torchrun with EPB_TRACE=1).

Each rank runs a few DeepSeek-V3 normal steps and LL steps; rank 0 prints the
intervals between its phase marks (see trace_mark() calls in csrc/)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ.setdefault("EPB_TRACE", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch
import torch.distributed as dist

import paper_2512_19849_b200 as epb
from paper_2512_19849_b200._lib import lib
from tests.helpers import bf16_random, make_routing, to_dev_bf16

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
H, E, K, T = 7168, 256, 8, 4096
g = np.random.default_rng(rank)
idx, w = make_routing(g, T, E, K)
x = to_dev_bf16(bf16_random(g, (T, H)))
topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
buf = epb.Buffer(dist.group.WORLD, epb.nvl_bytes_hint(T, H, world, K),
                 epb.Buffer.get_low_latency_rdma_size_hint(128, H, world, E, K), low_latency_mode=True)
y = torch.randn(E // world, world * 128, H, device="cuda").to(torch.bfloat16)
NAMES = {0: "start", 1: "arrive+counts", 2: "scan", 3: "post msgs", 4: "peers' msgs", 5: "plan published",
         6: "host publish", 7: "plan loaded", 9: "copies done", 10: "all arrived", 16: "combine start",
         17: "push done", 18: "barrier", 19: "reduce done", 24: "ll_disp start", 25: "bitmap", 26: "items done",
         27: "ticket", 28: "recv wait", 33: "ll_comb items", 34: "ll_comb wait"}


def show(label):
    tr = (C.c_int64 * 64)()
    lib.epb_trace(buf._rank.ctx, tr)
    ts = {i: tr[i] for i in range(64) if tr[i]}
    print(label, flush=True)
    for a, b in [(0, 10), (16, 19), (24, 28), (32, 35)]:
        keys = [k for k in sorted(ts) if a <= k <= b]
        if keys:
            t0 = ts[keys[0]]
            print("   " + "  ".join(f"{NAMES.get(k, k)}=+{(ts[k] - t0) / 1e3:.2f}us" for k in keys), flush=True)


for i in range(8):
    pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                         topk_idx=topk, topk_weights=wt)
    out, _, _ = buf.combine(rx, h, topk_weights=rtw)
torch.cuda.synchronize()
dist.barrier()
if rank == 0:
    show(f"normal (EP={world}, {T} tokens/rank)")
for i in range(8):
    recv, cnt, hd, _, _ = buf.low_latency_dispatch(x[:128].contiguous(), topk[:128].contiguous(), 128, E)
    o, _, _ = buf.low_latency_combine(y, topk[:128].contiguous(), wt[:128].contiguous(), hd)
torch.cuda.synchronize()
dist.barrier()
if rank == 0:
    show(f"low latency (EP={world}, 128 tokens/rank)")
buf.destroy()
dist.barrier()
dist.destroy_process_group()
