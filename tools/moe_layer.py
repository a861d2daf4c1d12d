"""Caller-side integration: an expert-parallel MoE layer on
the Buffer API — router -> dispatch -> grouped expert GEMMs -> combine — in the
two shapes DeepEP users run:

* prefill / training: normal mode (``get_dispatch_layout`` -> ``dispatch`` ->
  per-expert SwiGLU on the received rows -> ``combine``);
* decode: low-latency mode (FP8 ``low_latency_dispatch`` -> one batched GEMM
  per projection over the packed [L, R*Tmax, H] layout -> ``low_latency_combine``),
  optionally with ``return_recv_hook`` so a shared expert runs while the tokens
  are in flight, and captured in a CUDA graph.

The expert math is plain torch (cuBLAS); the communication is this package.
Run as a microbench:  python tools/moe_layer.py  (or under torchrun for EP>1).
"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import torch.nn.functional as F


class MoELayer:
    """Top-k routed SwiGLU experts, expert-parallel over the Buffer's ranks
    (experts [rank*L, (rank+1)*L) live here)."""

    def __init__(self, buf, hidden: int, ffn: int, num_experts: int, topk: int, seed: int = 0,
                 device: str = "cuda"):
        self.buf, self.H, self.F, self.E, self.k = buf, hidden, ffn, num_experts, topk
        self.R, self.rank = buf.group_size, buf.rank
        self.L = num_experts // self.R
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.router = (torch.randn(hidden, num_experts, generator=g) * hidden ** -0.5).to(device, torch.bfloat16)
        lo = self.rank * self.L
        w1 = torch.randn(num_experts, hidden, 2 * ffn, generator=g)[lo:lo + self.L] * hidden ** -0.5
        w2 = torch.randn(num_experts, ffn, hidden, generator=g)[lo:lo + self.L] * ffn ** -0.5
        self.w1 = w1.to(device, torch.bfloat16).contiguous()  # [L, H, 2F] (gate | up)
        self.w2 = w2.to(device, torch.bfloat16).contiguous()  # [L, F, H]
        self.shared = (torch.randn(hidden, hidden, generator=g) * hidden ** -0.5).to(device, torch.bfloat16)

    # -- routing -------------------------------------------------------------------
    def route(self, x):
        logits = (x @ self.router).float()
        w, idx = torch.topk(torch.softmax(logits, dim=-1), self.k, dim=-1)
        return idx.to(torch.int64), (w / w.sum(-1, keepdim=True)).to(torch.float32)

    def _experts(self, xb):
        """SwiGLU over a batch per local expert: xb [L, n, H] bf16 -> [L, n, H] bf16."""
        h = torch.bmm(xb, self.w1)
        h = F.silu(h[..., : self.F]) * h[..., self.F:]
        return torch.bmm(h, self.w2)

    # -- normal mode (prefill / training) -------------------------------------------
    def forward_normal(self, x, idx=None, w=None):
        if idx is None:
            idx, w = self.route(x)
        per_rank, _, per_exp, in_rank, _ = self.buf.get_dispatch_layout(idx, self.E)
        recv_x, recv_idx, recv_w, counts, handle, _ = self.buf.dispatch(
            x, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank, num_tokens_per_expert=per_exp,
            topk_idx=idx, topk_weights=w)
        # one padded batch per local expert (counts come from the dispatch, on the host)
        n = recv_x.shape[0]
        cap = max(1, max(counts))
        sel = recv_idx >= 0                                    # [n, k] (row, slot) pairs for my experts
        rows, slots = sel.nonzero(as_tuple=True)
        le = recv_idx[rows, slots]
        order = torch.argsort(le, stable=True)
        rows, slots, le = rows[order], slots[order], le[order]
        starts = torch.zeros(self.L + 1, dtype=torch.int64, device=x.device)
        starts[1:] = torch.cumsum(torch.bincount(le, minlength=self.L), 0)
        pos = torch.arange(le.numel(), device=x.device) - starts[le]
        xb = torch.zeros(self.L, cap, self.H, dtype=torch.bfloat16, device=x.device)
        xb[le, pos] = recv_x[rows]
        yb = self._experts(xb)
        # weight each (row, expert) output by its gate and sum per row (fp32), one bf16 rounding
        y = torch.zeros(n, self.H, dtype=torch.float32, device=x.device)
        y.index_add_(0, rows, yb[le, pos].float() * recv_w[rows, slots].unsqueeze(1))
        out, _, _ = self.buf.combine(y.to(torch.bfloat16), handle)
        return out

    # -- low-latency mode (decode) -----------------------------------------------------
    def forward_ll(self, x, idx, w, max_tokens: int, overlap: bool = False):
        (q, s), count, handle, _, hook = self.buf.low_latency_dispatch(
            x, idx, max_tokens, self.E, use_fp8=True, return_recv_hook=overlap)
        shared = x @ self.shared if overlap else None  # runs while the tokens are in flight
        if overlap:
            hook()
        xb = (q.float().view(self.L, -1, self.H // 128, 128) * s.unsqueeze(-1)).view(self.L, -1, self.H)
        yb = self._experts(xb.to(torch.bfloat16))
        out, _, _ = self.buf.low_latency_combine(yb, idx, w, handle)
        return out if shared is None else (out, shared)


def dense_reference(layer: MoELayer, x, idx, w, all_w1=None, all_w2=None):
    """Every expert on every token, no communication (single rank: all experts local)."""
    w1 = layer.w1 if all_w1 is None else all_w1
    w2 = layer.w2 if all_w2 is None else all_w2
    out = torch.zeros(x.shape[0], layer.H, dtype=torch.float32, device=x.device)
    for j in range(layer.k):
        e = idx[:, j]
        h = torch.bmm(x.unsqueeze(1), w1[e]).squeeze(1)
        h = F.silu(h[:, : layer.F]) * h[:, layer.F:]
        y = torch.bmm(h.unsqueeze(1), w2[e]).squeeze(1)
        out += y.float() * w[:, j:j + 1]
    return out.to(torch.bfloat16)


def main():
    import torch.distributed as dist
    import paper_2512_19849_b200 as epb
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
        group = dist.group.WORLD
    T, H, Fd, E, k, Tm = 4096, 7168, 2048, 256, 8, 128
    buf = epb.Buffer(group, epb.nvl_bytes_hint(T, H, world, k), epb.Buffer.get_low_latency_rdma_size_hint(
        Tm, H, world, E, num_topk=k), low_latency_mode=True)
    layer = MoELayer(buf, H, Fd, E, k, seed=1)
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    idx, w = layer.route(x)

    def timed(fn, n=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3

    t_layer = timed(lambda: layer.forward_normal(x, idx, w))
    xd = x[:Tm].contiguous()
    idd, wd = idx[:Tm].contiguous(), w[:Tm].contiguous()
    t_ll = timed(lambda: layer.forward_ll(xd, idd, wd, Tm))
    t_ll_ov = timed(lambda: layer.forward_ll(xd, idd, wd, Tm, overlap=True))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        layer.forward_ll(xd, idd, wd, Tm)
        with torch.cuda.graph(g, stream=s):
            layer.forward_ll(xd, idd, wd, Tm)
    torch.cuda.current_stream().wait_stream(s)
    t_graph = timed(g.replay, 50)
    if rank == 0:
        print(f"MoE layer EP={world}: prefill {T} tok x H={H}, F={Fd}, {E} experts, top-{k}: {t_layer:.0f} us/forward; "
              f"decode {Tm} tok (FP8 LL): eager {t_ll:.0f} us, with recv hook + shared expert {t_ll_ov:.0f} us, "
              f"CUDA graph {t_graph:.0f} us", flush=True)
    buf.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
