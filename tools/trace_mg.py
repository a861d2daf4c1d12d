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
NAMES = {2: "gather start", 0: "start", 1: "arrive+counts", 3: "post msgs", 4: "peers' msgs", 5: "plan published",
         6: "host publish", 7: "plan loaded", 9: "copies done", 10: "all arrived", 15: "combine entry", 16: "combine start",
         17: "push done", 18: "barrier", 19: "reduce done", 24: "ll_disp start", 25: "bitmap", 26: "items done",
         27: "ticket", 28: "recv wait", 29: "ll_disp last block done", 32: "ll_comb start", 33: "ll_comb items", 34: "ll_comb wait", 35: "ll_comb last block done", 22: "consumers done (max)", **{40 + w: f"wave{w} ready" for w in range(8)}, **{48 + w: f"wave{w} pushed(b0)" for w in range(8)}, 11: "last block copy start", 12: "last block copies done", 20: "last block reduce done", 21: "last block reduce start"}


def snap():
    tr = (C.c_int64 * 64)()
    lib.epb_trace(buf._rank.ctx, tr)
    return {i: tr[i] for i in range(64) if tr[i]}


def show(label, snaps):
    """Median over calls of each mark's offset from the first mark of its group."""
    import statistics
    print(label, flush=True)
    for grp in [range(0, 13), list(range(15, 23)) + list(range(40, 56)), range(24, 30), range(32, 36)]:
        offs = {}
        for ts in snaps:
            keys = [k for k in sorted(ts) if k in grp]
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
    dist.barrier()
    if i >= 5:
        snaps.append(snap())
if rank == 0:
    show(f"normal (EP={world}, {T} tokens/rank), median of 30 calls", snaps)
snaps = []
for i in range(35):
    recv, cnt, hd, _, _ = buf.low_latency_dispatch(x[:128].contiguous(), topk[:128].contiguous(), 128, E)
    o, _, _ = buf.low_latency_combine(y, topk[:128].contiguous(), wt[:128].contiguous(), hd)
    torch.cuda.synchronize()
    dist.barrier()
    if i >= 5:
        snaps.append({k: v for k, v in snap().items() if k >= 24})
if rank == 0:
    show(f"low latency (EP={world}, 128 tokens/rank), median of 30 calls", snaps)
buf.destroy()
dist.barrier()
dist.destroy_process_group()
