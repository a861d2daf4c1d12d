"""2+ GPU check of the HT proxy transport at DS-V3 size (torchrun): the proxy
Buffer's dispatch/combine outputs must equal the NVLink Buffer's bit for bit;
prints per-call device times."""
import os, sys, time
os.environ.setdefault("EPB_TIMEOUT_S", "10")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
import paper_2512_19849_b200 as epb
from tests.helpers import bf16_random, make_routing
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
H, E, K = 7168, 256, 8
ref = epb.Buffer(dist.group.WORLD, epb.nvl_bytes_hint(T, H, world, K, 2), 0, num_recv_slots=2)
buf = epb.Buffer(dist.group.WORLD, epb.nvl_bytes_hint(T, H, world, K, 2, ht_proxy=True), 0, num_recv_slots=2,
                 fifo_channels=8, proxy_threads=4, ht_transport="proxy")
g = np.random.default_rng(rank)
idx, w = make_routing(g, T, E, K)
x = torch.from_numpy(bf16_random(g, (T, H)).view(np.int16)).view(torch.bfloat16).cuda()
idx_t, w_t = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ok = True
side = torch.cuda.Stream() if os.environ.get("SIDE") else None
if side is not None:
    torch.cuda.set_stream(side)
import bench as _bench
for it in range(4):
    outs = {}
    for name, b in (("nvlink", ref), ("proxy", buf)):
        pr, _, pe, ir, _ = b.get_dispatch_layout(idx_t, E)
        dist.barrier(); torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        flush.zero_()
        e[0].record()
        try:
            rx, rti, rtw, _, h, _ = b.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir,
                                               num_tokens_per_expert=pe, topk_idx=idx_t, topk_weights=w_t)
            if os.environ.get("SYNC_AFTER_DISPATCH"):
                torch.cuda.synchronize()
        except Exception:
            if name == "proxy":
                _bench._proxy_diag(b, rank)
            raise
        if name == "proxy" and os.environ.get("SYNC_AFTER_DISPATCH"):
            try:
                torch.cuda.synchronize()
                b._g.check_device_error()
            except Exception:
                _bench._proxy_diag(b, rank)
                raise
        e[1].record()
        flush.zero_()
        y = rx if it % 2 == 0 else rx.clone()  # in place / staged
        if name == "nvlink" and os.environ.get("REF_MODE") == "push":
            y = rx.clone()
        if name == "nvlink" and os.environ.get("REF_MODE") == "nocombine":
            out, ow = rx, rtw
        else:
            out, ow, _ = b.combine(y, h, topk_weights=rtw)
        e[2].record()
        torch.cuda.synchronize()
        outs[name] = (rx.clone(), rtw.clone(), out, ow)
        print(f"rank {rank} it {it} {name}: dispatch {e[0].elapsed_time(e[1])*1e3:.0f} us, "
              f"combine {e[1].elapsed_time(e[2])*1e3:.0f} us", flush=True)
    same = all(torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a,
                           b_.view(torch.int16) if b_.dtype == torch.bfloat16 else b_)
               for a, b_ in zip(outs["nvlink"], outs["proxy"]))
    ok &= same
    print(f"rank {rank} it {it}: proxy == nvlink: {same}", flush=True)
for b in (ref, buf):
    b._g.check_device_error()
    b.destroy()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
