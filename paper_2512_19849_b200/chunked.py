"""Host side of the chunked-ring transport (``ht_transport="ring"``; SURVEY
8(f) f1, csrc/chunked.cu).

DeepEP's normal-mode flow with bounded buffers: the count exchange runs first
(``epb_dispatch_notify``: handle matrices, send_head, host counts), the host
sizes the receive tensors from the notified counts, then the ring kernel moves
the rows through the per-(source, lane) rings (SPEC.md:409-413 RingChannel,
:436-444 dispatch_ht).  The combine sends the expert outputs back through the
mirror rings and reduces at the source in canonical order (SPEC.md:446-454,
:477).  Outputs and handle match the direct transport (``Buffer.dispatch``)
bit for bit; only the memory bound and the data path differ.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import torch

from . import _lib as L
from ._lib import check, lib, raw_stream
from .errors import ConfigError


def ring_layout(rank, hidden: int, num_topk: int, lanes: int = 0, n_local: int = 1) -> L.RingLayout:
    out = L.RingLayout()
    check(lib.epb_ring_layout(rank.ctx, int(hidden), int(num_topk), int(lanes), int(n_local), C.byref(out)))
    return out


def _ctxs(ranks):
    return (C.c_void_p * len(ranks))(*[r.ctx.value for r in ranks])


def _ptr(t: Optional[torch.Tensor]) -> int:
    return 0 if t is None else t.data_ptr()


def ring_dispatch(ranks, xs, x_scales, in_ranks, per_experts, topk_idxs, topk_ws, expert_alignment: int,
                  channels: int, timeout_s: float, lanes: int = 0):
    """Per rank: (recv_x | (recv_x, scales), recv_topk_idx, recv_topk_weights,
    num_recv_tokens_per_expert_list, handle) — the shapes of Buffer.dispatch."""
    n = len(ranks)
    R = ranks[0].world
    Cn = int(channels)
    args = (L.DispatchArgs * n)()
    keep = []
    for i in range(n):
        x = xs[i].contiguous()
        fp8 = x.dtype == torch.float8_e4m3fn
        if fp8 and x_scales[i] is None:
            raise ConfigError("FP8 dispatch needs scales")
        if not fp8 and x.dtype != torch.bfloat16:
            raise ConfigError("dispatch expects bf16 x or an (fp8, scales) tuple")
        sc = x_scales[i].contiguous() if fp8 else None
        T, H = x.shape
        ir = in_ranks[i].contiguous()
        if ir.dtype != torch.bool or tuple(ir.shape) != (T, R):
            raise ConfigError("is_token_in_rank must be bool [num_tokens, num_ranks]")
        ti = topk_idxs[i].contiguous() if topk_idxs[i] is not None else None
        tw = topk_ws[i].to(torch.float32).contiguous() if (ti is not None and topk_ws[i] is not None) else None
        pe = per_experts[i].contiguous() if per_experts[i] is not None else None
        if ti is not None and pe is None:
            raise ConfigError("num_tokens_per_expert is required with topk_idx")
        hbuf = torch.empty(R * R + 2 * R * Cn + T * R, dtype=torch.int32, device=x.device)
        a = args[i]
        a.x, a.x_scales = x.data_ptr(), _ptr(sc)
        a.hidden, a.elem_bytes, a.num_scales = H, 1 if fp8 else 2, (sc.shape[1] if sc is not None else 0)
        a.topk_idx, a.topk_weights = _ptr(ti), _ptr(tw)
        a.num_topk = ti.shape[1] if ti is not None else 0
        a.is_token_in_rank = ir.data_ptr()
        a.num_tokens_per_expert = _ptr(pe)
        a.num_tokens, a.num_experts = T, (pe.numel() if pe is not None else 0)
        a.expert_alignment = max(1, int(expert_alignment))
        a.recv_slot = 0
        base = hbuf.data_ptr()
        a.rank_prefix_matrix = base
        a.channel_prefix_matrix = base + 4 * R * R
        a.recv_channel_prefix_matrix = base + 4 * (R * R + R * Cn)
        a.send_head = base + 4 * (R * R + 2 * R * Cn)
        keep.append((x, sc, ir, ti, tw, pe, hbuf))
    ctxs = _ctxs(ranks)
    stream = raw_stream()
    check(lib.epb_dispatch_notify(ctxs, n, args, Cn, stream))
    counts = []
    for i in range(n):
        E = args[i].num_experts
        Lx = E // R if E else 0
        nrecv = C.c_int64()
        per = (C.c_int32 * max(1, Lx))()
        check(lib.epb_wait_notify(ranks[i].ctx, C.byref(nrecv), per if Lx else None, Lx, float(timeout_s)))
        counts.append((nrecv.value, [per[j] for j in range(Lx)] if Lx else None))
    rargs = (L.RingDispatchArgs * n)()
    outs = []
    for i in range(n):
        x, sc, ir, ti, tw, pe, hbuf = keep[i]
        a, N = args[i], counts[i][0]
        dev = x.device
        recv_x = torch.empty((N, a.hidden), dtype=x.dtype, device=dev)
        recv_sc = torch.empty((N, a.num_scales), dtype=torch.float32, device=dev) if sc is not None else None
        recv_ti = torch.empty((N, a.num_topk), dtype=torch.int64, device=dev) if ti is not None else None
        recv_tw = torch.empty((N, a.num_topk), dtype=torch.float32, device=dev) if tw is not None else None
        recv_src = torch.empty((N,), dtype=torch.int32, device=dev)
        r = rargs[i]
        r.x, r.x_scales, r.hidden, r.elem_bytes, r.num_scales = a.x, a.x_scales, a.hidden, a.elem_bytes, a.num_scales
        r.topk_idx, r.topk_weights, r.num_topk = a.topk_idx, a.topk_weights, a.num_topk
        r.num_tokens, r.num_experts = a.num_tokens, a.num_experts
        r.rank_prefix_matrix, r.recv_channel_prefix_matrix = a.rank_prefix_matrix, a.recv_channel_prefix_matrix
        r.send_head, r.num_channels = a.send_head, Cn
        r.recv_x, r.recv_x_scales = recv_x.data_ptr(), _ptr(recv_sc)
        r.recv_topk_idx, r.recv_topk_weights, r.recv_src_idx = _ptr(recv_ti), _ptr(recv_tw), recv_src.data_ptr()
        r.num_recv = N
        T = a.num_tokens
        rpm = hbuf[: R * R].view(R, R)
        cpm = hbuf[R * R: R * R + R * Cn].view(R, Cn)
        rcpm = hbuf[R * R + R * Cn: R * R + 2 * R * Cn].view(R, Cn)
        send_head = hbuf[R * R + 2 * R * Cn:].view(T, R)
        handle = (rpm, cpm, rcpm, recv_src, ir, send_head)
        px = (recv_x, recv_sc) if sc is not None else recv_x
        outs.append((px, recv_ti, recv_tw, counts[i][1], handle))
    check(lib.epb_ring_dispatch(ctxs, n, rargs, int(lanes), stream))
    return outs


def ring_combine(ranks, xs: Sequence[torch.Tensor], handles, topk_ws, lanes: int = 0) -> List[tuple]:
    """Per rank: (combined_x, combined_topk_weights | None), as Buffer.combine."""
    n = len(ranks)
    args = (L.RingCombineArgs * n)()
    outs, keep = [], []
    for i in range(n):
        x = xs[i].contiguous()
        if x.dtype != torch.bfloat16:
            raise ConfigError("combine expects bf16 rows")
        h = handles[i]
        rpm, rcpm, recv_src, send_head = h[0], h[2], h[3], h[5]
        if x.shape[0] != recv_src.numel():
            raise ConfigError("combine input rows do not match the dispatch handle")
        T = send_head.shape[0]
        tw = topk_ws[i].to(torch.float32).contiguous() if topk_ws[i] is not None else None
        k = tw.shape[1] if tw is not None else 0
        out = torch.empty((T, x.shape[1]), dtype=torch.bfloat16, device=x.device)
        out_w = torch.empty((T, k), dtype=torch.float32, device=x.device) if tw is not None else None
        a = args[i]
        a.x, a.topk_weights = x.data_ptr(), _ptr(tw)
        a.num_recv, a.hidden, a.num_topk = x.shape[0], x.shape[1], k
        a.rank_prefix_matrix, a.recv_channel_prefix_matrix = rpm.data_ptr(), rcpm.data_ptr()
        a.send_head, a.num_channels, a.num_tokens = send_head.data_ptr(), rcpm.shape[1], T
        a.combined_x, a.combined_topk_weights = out.data_ptr(), _ptr(out_w)
        keep.append((x, tw))
        outs.append((out, out_w))
    check(lib.epb_ring_combine(_ctxs(ranks), n, args, int(lanes), raw_stream()))
    return outs
