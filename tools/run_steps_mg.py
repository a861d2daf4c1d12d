"""A few DeepSeek-V3 normal-mode steps (layout -> dispatch -> combine) on every
rank of a torchrun job, for single-pass ncu captures of the NVLink counters:

    ncu --target-processes all --replay-mode kernel --cache-control none \
        --clock-control none --metrics gpu__time_duration.sum,nvltx__bytes.sum,... \
        torchrun --nproc-per-node N tools/run_steps_mg.py [steps]

Only metric sets that fit in ONE pass work: a replayed dispatch/combine would
wait for peer messages that ncu's memory restore erased (EPB_TIMEOUT_S bounds
that wait).
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch
import torch.distributed as dist

import paper_2512_19849_b200 as epb
from tests.helpers import bf16_random, make_routing, to_dev_bf16

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
H, E, K, T = 7168, 256, 8, 4096
g = np.random.default_rng(rank)
idx, w = make_routing(g, T, E, K)
x = to_dev_bf16(bf16_random(g, (T, H)))
topk, wt = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
buf = epb.Buffer(dist.group.WORLD, epb.nvl_bytes_hint(T, H, world, K))
for _ in range(steps):
    pr, _, pe, ir, _ = buf.get_dispatch_layout(topk, E)
    rx, rti, rtw, _, h, _ = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                         topk_idx=topk, topk_weights=wt)
    out, _, _ = buf.combine(rx, h, topk_weights=rtw)
torch.cuda.synchronize()
m = torch.zeros(T, world, dtype=torch.bool, device="cuda")
m.scatter_(1, topk // (E // world), True)
m[:, rank] = False
print(f"rank {rank}: remote rows per step {int(m.sum())} = {int(m.sum()) * 2 * H / 1e6:.1f} MB per direction",
      flush=True)
buf.destroy()
dist.barrier()
dist.destroy_process_group()
