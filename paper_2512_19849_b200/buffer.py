"""DeepEP-compatible ``Buffer`` for the B200 EP dispatch/combine path.

The paper claims drop-in compatibility with DeepEP's Python API
(PAPER.md:98); that API is not vendored in the reference, so the
signatures below follow DeepEP's public ``deep_ep.Buffer``.
Every method is a thin host wrapper around the C ABI (include/epb.h):

* ``Buffer.__init__``        -> epb_create + CUDA-IPC handle all-gather + epb_open_peers
* ``get_dispatch_layout``    -> epb_get_dispatch_layout        (SPEC.md:416-424 plan_dedup)
* ``dispatch``               -> epb_notify_dispatch, epb_wait_notify, epb_dispatch
* ``combine``                -> epb_combine
* ``low_latency_dispatch``   -> epb_ll_dispatch
* ``low_latency_combine``    -> epb_ll_combine

``torch.distributed`` is used once, at construction, to exchange IPC handles;
nothing on the data path calls a collective.

``LocalGroup`` runs R ranks inside one process on one GPU (each rank gets its
own symmetric region; "peers" are plain device pointers) and launches every
phase as ONE kernel over all ranks, so cross-rank waits never span separate
launches.  It exists for single-GPU parity tests of multi-rank routing; it is
not a performance configuration.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import Callable, List, Optional, Sequence, Tuple, Union

import torch

from . import _lib as L
from ._lib import check, lib, ptr
from .errors import ConfigError, ProtocolViolation, UnsupportedOperation

_DEFAULT_TIMEOUT_S = float(os.environ.get("EPB_TIMEOUT_S", "30"))


def _device_sms() -> int:
    n = lib.epb_num_sms()
    return n if n > 0 else 148


class EventOverlap:
    """DeepEP's EventOverlap: an optional CUDA event plus tensors kept alive."""

    def __init__(self, event: Optional[torch.cuda.Event] = None, extra_tensors=None):
        self.event = event
        self.extra_tensors = extra_tensors

    def current_stream_wait(self) -> None:
        if self.event is not None:
            torch.cuda.current_stream().wait_event(self.event)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.current_stream_wait()


class Config:
    """DeepEP-style performance config.  ``num_sms`` is the grid width of the
    dispatch (one channel per block) and combine kernels; the chunk sizes are
    accepted for API compatibility (this path pushes whole rows directly into
    final receive slots, so there is no chunked ring to size)."""

    def __init__(self, num_sms: Optional[int] = None, num_max_nvl_chunked_send_tokens: int = 6,
                 num_max_nvl_chunked_recv_tokens: int = 256, num_max_rdma_chunked_send_tokens: int = 6,
                 num_max_rdma_chunked_recv_tokens: int = 256):
        self.num_sms = int(num_sms) if num_sms else 0
        self.num_max_nvl_chunked_send_tokens = num_max_nvl_chunked_send_tokens
        self.num_max_nvl_chunked_recv_tokens = num_max_nvl_chunked_recv_tokens
        self.num_max_rdma_chunked_send_tokens = num_max_rdma_chunked_send_tokens
        self.num_max_rdma_chunked_recv_tokens = num_max_rdma_chunked_recv_tokens

    def resolved_sms(self) -> int:
        return min(self.num_sms or _device_sms(), L.MAX_CHANNELS)

    def get_nvl_buffer_size_hint(self, hidden_bytes: int, num_ranks: int, num_tokens: int = 4096,
                                 num_topk: int = 8, num_slots: int = 3) -> int:
        return nvl_bytes_hint(num_tokens, hidden_bytes // 2, num_ranks, num_topk, num_slots)


def nvl_bytes_hint(num_tokens: int, hidden: int, num_ranks: int, num_topk: int = 8, num_slots: int = 3) -> int:
    """Arena bytes so that the worst case (every token to every rank) fits:
    ``num_slots`` receive slots + 2 combine staging buffers of R*T rows."""
    rows = num_ranks * num_tokens
    per_row = 2 * hidden + 4 * (hidden // 128) + 12 * num_topk + 4
    comb_row = 2 * hidden + 4 * num_topk
    return rows * (num_slots * per_row + 2 * comb_row) + 256 * (6 * num_slots + 6) + (1 << 20)


class _SlotMemory:
    """``__cuda_array_interface__`` view of one receive slot.  The torch tensor
    built from it keeps this object alive; when the last view of the slot dies
    the slot returns to its rank's free list."""

    def __init__(self, addr: int, nbytes: int, release: Optional[Callable[[], None]]):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (addr, False), "version": 3, "strides": None,
            "stream": None,
        }
        self._release = release

    def __del__(self):
        if self._release is not None:
            self._release()


class _Rank:
    """Native state of one EP rank (the epb_t* and its receive-slot leases)."""

    def __init__(self, rank: int, world: int, nvl_bytes: int, ll_bytes: int, num_recv_slots: int,
                 fifo_channels: int, fifo_capacity: int, proxy_threads: int):
        self.rank, self.world = rank, world
        self.device = torch.device("cuda", torch.cuda.current_device())
        cfg = L.Config(nvl_bytes, ll_bytes, num_recv_slots, fifo_channels, fifo_capacity, proxy_threads)
        ctx = C.c_void_p()
        check(lib.epb_create(C.byref(ctx), rank, world, C.byref(cfg)))
        self.ctx = ctx
        self.cfg = cfg
        base, nbytes = C.c_void_p(), C.c_size_t()
        check(lib.epb_region(ctx, C.byref(base), C.byref(nbytes)))
        self.base, self.region_bytes = base.value, nbytes.value
        self.num_slots = max(1, num_recv_slots)
        # the last slot is the scratch slot used (with a copy-out) when every
        # leasable slot is still referenced by user tensors
        self.scratch_slot = self.num_slots - 1
        self._free = list(range(self.num_slots - 1))
        self._lock = threading.Lock()
        self._layouts = {}
        self.proxy_running = False

    # -- receive slots -----------------------------------------------------
    def recv_layout(self, hidden: int, num_topk: int) -> L.RecvLayout:
        key = (hidden, num_topk)
        lay = self._layouts.get(key)
        if lay is None:
            lay = L.RecvLayout()
            check(lib.epb_recv_layout(self.ctx, hidden, num_topk, C.byref(lay)))
            self._layouts[key] = lay
        return lay

    def lease_slot(self) -> Tuple[int, bool]:
        with self._lock:
            if self._free:
                return self._free.pop(0), False
        return self.scratch_slot, True

    def _release_slot(self, slot: int) -> None:
        with self._lock:
            self._free.append(slot)

    def slot_storage(self, lay: L.RecvLayout, slot: int, leased: bool) -> torch.Tensor:
        addr = self.base + lay.slot0_off + slot * lay.slot_bytes
        rel = (lambda s=slot: self._release_slot(s)) if leased else None
        return torch.as_tensor(_SlotMemory(addr, lay.slot_bytes, rel), device=self.device)

    def destroy(self) -> None:
        if self.ctx:
            lib.epb_destroy(self.ctx)
            self.ctx = None


def _ctx_array(ranks: Sequence[_Rank]):
    return (C.c_void_p * len(ranks))(*[r.ctx.value for r in ranks])


def _as_tuple_x(x):
    if isinstance(x, tuple):
        x_data, x_scales = x
        if x_data.dtype != torch.float8_e4m3fn:
            raise ConfigError("FP8 dispatch expects (x: float8_e4m3fn [T, H], scales: float32 [T, H/128])")
        if x_scales.dtype != torch.float32 or x_scales.dim() != 2:
            raise ConfigError("FP8 scales must be float32 [T, H/128]")
        return x_data.contiguous(), x_scales.contiguous(), 1
    if x.dtype != torch.bfloat16:
        raise ConfigError("dispatch expects bf16 x or an (fp8, scales) tuple")
    return x.contiguous(), None, 2


class _Group:
    """List-based implementation shared by Buffer (1 rank) and LocalGroup (R ranks)."""

    def __init__(self, ranks: List[_Rank], num_experts_hint: int = 0):
        self.ranks = ranks
        self.world = ranks[0].world
        self.timeout_s = _DEFAULT_TIMEOUT_S
        self._ctxs = _ctx_array(ranks)
        # optional per-launch CUDA-event records [(name, start, end)] for benchmarks
        self.prof: Optional[list] = None

    def _launch(self, name: str, fn) -> None:
        if self.prof is None:
            check(fn())
            return
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        check(fn())
        e.record()
        self.prof.append((name, s, e))

    # -- layout ------------------------------------------------------------
    def get_dispatch_layout(self, topk_idx_list: Sequence[torch.Tensor], num_experts: int):
        out = []
        stream = torch.cuda.current_stream().cuda_stream
        for topk_idx in topk_idx_list:
            if topk_idx.dtype != torch.int64 or topk_idx.dim() != 2:
                raise ConfigError("topk_idx must be int64 [num_tokens, num_topk]")
            topk_idx = topk_idx.contiguous()
            T, k = topk_idx.shape
            dev = topk_idx.device
            per_rank = torch.empty(self.world, dtype=torch.int32, device=dev)
            per_expert = torch.empty(num_experts, dtype=torch.int32, device=dev)
            in_rank = torch.empty((T, self.world), dtype=torch.bool, device=dev)
            self._launch("layout", lambda: lib.epb_get_dispatch_layout(
                ptr(topk_idx), T, k, num_experts, self.world, ptr(per_rank), ptr(per_expert), ptr(in_rank), stream))
            out.append((per_rank, None, per_expert, in_rank))
        return out

    # -- normal dispatch ---------------------------------------------------
    def dispatch(self, xs, handles, is_token_in_ranks, num_tokens_per_experts, topk_idxs, topk_weights_list,
                 expert_alignment: int, config: Optional[Config]):
        n = len(self.ranks)
        R = self.world
        cfg = config or Config()
        C_ = cfg.resolved_sms()
        stream = torch.cuda.current_stream().cuda_stream
        cached = handles[0] is not None
        args = (L.DispatchArgs * n)()
        keep = []
        per_rank_state = []
        for i, rk in enumerate(self.ranks):
            x, x_scales, elem = _as_tuple_x(xs[i])
            T, H = x.shape
            if cached:
                in_rank = handles[i][4]
                topk_idx = topk_weights = per_expert = None
            else:
                in_rank = is_token_in_ranks[i]
                topk_idx = topk_idxs[i]
                topk_weights = topk_weights_list[i]
                per_expert = num_tokens_per_experts[i]
            if in_rank is None or in_rank.shape != (T, R) or in_rank.dtype != torch.bool:
                raise ConfigError("is_token_in_rank must be bool [num_tokens, num_ranks]")
            in_rank = in_rank.contiguous()
            k = 0
            E = 0
            if topk_idx is not None:
                topk_idx = topk_idx.contiguous()
                k = topk_idx.shape[1]
                if topk_weights is not None:
                    topk_weights = topk_weights.to(torch.float32).contiguous()
            if per_expert is not None:
                E = per_expert.numel()
            elif topk_idx is not None:
                raise ConfigError("num_tokens_per_expert is required with topk_idx")
            lay = rk.recv_layout(H, k)
            slot, copy_out = rk.lease_slot()
            dev = x.device
            rpm = torch.empty((R, R), dtype=torch.int32, device=dev)
            cpm = torch.empty((R, C_), dtype=torch.int32, device=dev)
            rcpm = torch.empty((R, C_), dtype=torch.int32, device=dev)
            send_head = torch.empty((T, R), dtype=torch.int32, device=dev)
            a = args[i]
            a.x, a.x_scales = ptr(x), ptr(x_scales)
            a.hidden, a.elem_bytes = H, elem
            a.num_scales = 0 if x_scales is None else x_scales.shape[1]
            a.topk_idx, a.topk_weights, a.num_topk = ptr(topk_idx), ptr(topk_weights), k
            a.is_token_in_rank = ptr(in_rank)
            a.num_tokens_per_expert = ptr(per_expert)
            a.num_tokens, a.num_experts, a.expert_alignment = T, E, max(1, int(expert_alignment))
            a.recv_slot = slot
            a.rank_prefix_matrix, a.channel_prefix_matrix = ptr(rpm), ptr(cpm)
            a.recv_channel_prefix_matrix, a.send_head = ptr(rcpm), ptr(send_head)
            keep.append((x, x_scales, topk_idx, topk_weights, in_rank, per_expert))
            per_rank_state.append(dict(x=x, x_scales=x_scales, elem=elem, T=T, H=H, k=k, E=E, lay=lay, slot=slot,
                                       copy_out=copy_out, rpm=rpm, cpm=cpm, rcpm=rcpm, send_head=send_head,
                                       in_rank=in_rank, topk_idx=topk_idx, topk_weights=topk_weights))
        try:
            self._launch("notify", lambda: lib.epb_notify_dispatch(self._ctxs, n, args, C_, stream))
            # the dispatch kernel reads its plan (peer slots, row bases) from device
            # memory written by notify, so it is enqueued before the host waits for
            # the receive counts; if notify flagged an error the kernel moves no data
            self._launch("dispatch", lambda: lib.epb_dispatch(self._ctxs, n, args, C_, stream))
            for i, rk in enumerate(self.ranks):
                st = per_rank_state[i]
                Lx = st["E"] // R if st["E"] else 0
                nrecv = C.c_int64()
                per_exp = (C.c_int32 * max(1, Lx))()
                check(lib.epb_wait_notify(rk.ctx, C.byref(nrecv), per_exp if Lx else None, Lx, self.timeout_s))
                st["num_recv"] = nrecv.value
                st["per_expert_list"] = [int(per_exp[j]) for j in range(Lx)] if Lx else None
        except Exception:
            for st, rk in zip(per_rank_state, self.ranks):
                if not st["copy_out"]:
                    rk._release_slot(st["slot"])
            raise
        results = []
        for i, rk in enumerate(self.ranks):
            st = per_rank_state[i]
            lay, N, H, k = st["lay"], st["num_recv"], st["H"], st["k"]
            mem = rk.slot_storage(lay, st["slot"], leased=not st["copy_out"])
            row_bytes = H * st["elem"]
            xdt = torch.bfloat16 if st["elem"] == 2 else torch.float8_e4m3fn
            recv_x = mem[lay.off_x: lay.off_x + N * row_bytes].view(xdt).view(N, H)
            recv_scales = None
            if st["x_scales"] is not None:
                S = st["x_scales"].shape[1]
                recv_scales = mem[lay.off_scales: lay.off_scales + N * S * 4].view(torch.float32).view(N, S)
            recv_src_idx = mem[lay.off_src_idx: lay.off_src_idx + N * 4].view(torch.int32)
            recv_topk_idx = recv_topk_w = None
            if st["topk_idx"] is not None:
                recv_topk_idx = mem[lay.off_topk_idx: lay.off_topk_idx + N * k * 8].view(torch.int64).view(N, k)
                if st["topk_weights"] is not None:
                    recv_topk_w = mem[lay.off_topk_w: lay.off_topk_w + N * k * 4].view(torch.float32).view(N, k)
            if st["copy_out"]:
                recv_x = recv_x.clone()
                recv_src_idx = recv_src_idx.clone()
                recv_scales = None if recv_scales is None else recv_scales.clone()
                recv_topk_idx = None if recv_topk_idx is None else recv_topk_idx.clone()
                recv_topk_w = None if recv_topk_w is None else recv_topk_w.clone()
            del mem
            handle = (st["rpm"], st["cpm"], st["rcpm"], recv_src_idx, st["in_rank"], st["send_head"])
            out_x = (recv_x, recv_scales) if recv_scales is not None else recv_x
            results.append((out_x, recv_topk_idx, recv_topk_w, st["per_expert_list"], handle))
        return results

    # -- normal combine ----------------------------------------------------
    def combine(self, xs, handles, topk_weights_list, config: Optional[Config]):
        n = len(self.ranks)
        cfg = config or Config()
        stream = torch.cuda.current_stream().cuda_stream
        args = (L.CombineArgs * n)()
        outs, keep = [], []
        for i in range(n):
            x = xs[i]
            if x.dtype != torch.bfloat16 or x.dim() != 2:
                raise ConfigError("combine expects bf16 x [num_recv_tokens, hidden]")
            x = x.contiguous()
            rpm, _cpm, _rcpm, recv_src_idx, in_rank, send_head = handles[i]
            N, H = x.shape
            if N != recv_src_idx.numel():
                raise ProtocolViolation("combine input rows do not match the dispatch handle")
            T = in_rank.shape[0]
            w = topk_weights_list[i] if topk_weights_list is not None else None
            k = 0
            if w is not None:
                w = w.to(torch.float32).contiguous()
                k = w.shape[1]
            out = torch.empty((T, H), dtype=torch.bfloat16, device=x.device)
            out_w = torch.empty((T, k), dtype=torch.float32, device=x.device) if w is not None else None
            a = args[i]
            a.x, a.topk_weights, a.num_recv, a.hidden, a.num_topk = ptr(x), ptr(w), N, H, k
            a.rank_prefix_matrix, a.is_token_in_rank, a.send_head = ptr(rpm), ptr(in_rank), ptr(send_head)
            a.num_tokens, a.combined_x, a.combined_topk_weights = T, ptr(out), ptr(out_w)
            keep.append((x, w))
            outs.append((out, out_w))
        self._launch("combine", lambda: lib.epb_combine(self._ctxs, n, args, cfg.resolved_sms(), stream))
        return outs

    # -- low latency -------------------------------------------------------
    def ll_dispatch(self, xs, topk_idxs, num_max_dispatch_tokens_per_rank: int, num_experts: int, use_fp8: bool,
                    round_scale: bool, return_recv_hook: bool, use_proxy: bool):
        n = len(self.ranks)
        R = self.world
        if num_experts % R:
            raise ConfigError("num_experts must be a multiple of the number of ranks")
        Lx = num_experts // R
        Tm = int(num_max_dispatch_tokens_per_rank)
        stream = torch.cuda.current_stream().cuda_stream
        args = (L.LLDispatchArgs * n)()
        res, keep = [], []
        for i in range(n):
            x = xs[i]
            if x.dtype != torch.bfloat16 or x.dim() != 2:
                raise ConfigError("low_latency_dispatch expects bf16 x [num_tokens, hidden]")
            x = x.contiguous()
            topk_idx = topk_idxs[i].contiguous()
            T, H = x.shape
            k = topk_idx.shape[1]
            if T > Tm:
                raise ConfigError("num_tokens exceeds num_max_dispatch_tokens_per_rank")
            dev = x.device
            S = H // 128
            xdt = torch.float8_e4m3fn if use_fp8 else torch.bfloat16
            packed_x = torch.empty((Lx, R * Tm, H), dtype=xdt, device=dev)
            packed_s = (torch.empty((Lx, S, R * Tm), dtype=torch.float32, device=dev) if use_fp8 else None)
            count = torch.empty((Lx,), dtype=torch.int32, device=dev)
            src_info = torch.empty((Lx, R * Tm), dtype=torch.int32, device=dev)
            layout_range = torch.empty((Lx, R), dtype=torch.int64, device=dev)
            route = torch.empty((Lx, R * Tm), dtype=torch.int32, device=dev)
            comb_slot = torch.empty((T, k), dtype=torch.int32, device=dev)
            a = args[i]
            a.x, a.topk_idx, a.num_tokens, a.num_topk, a.hidden = ptr(x), ptr(topk_idx), T, k, H
            a.num_experts, a.max_tokens, a.use_fp8, a.round_scale = num_experts, Tm, int(use_fp8), int(round_scale)
            a.packed_recv_x, a.packed_recv_x_scales = ptr(packed_x), ptr(packed_s)
            a.packed_recv_count, a.packed_recv_src_info = ptr(count), ptr(src_info)
            a.packed_recv_layout_range, a.recv_route, a.comb_slot = ptr(layout_range), ptr(route), ptr(comb_slot)
            a.phases = 1 if return_recv_hook else 3
            a.use_proxy = int(use_proxy)
            keep.append((x, topk_idx))
            handle = (src_info, layout_range, Tm, H, num_experts, route, comb_slot, count, k, bool(use_proxy))
            recv = (packed_x, packed_s.transpose(1, 2)) if use_fp8 else packed_x
            res.append((recv, count, handle))
        self._launch("ll_dispatch", lambda: lib.epb_ll_dispatch(self._ctxs, n, args, _device_sms(), stream))
        hook = None
        if return_recv_hook:
            def hook(args=args, keep=keep):
                for i in range(n):
                    args[i].phases = 2
                check(lib.epb_ll_dispatch(self._ctxs, n, args, _device_sms(), torch.cuda.current_stream().cuda_stream))
        return res, hook

    def ll_combine(self, xs, topk_idxs, topk_weights_list, handles, return_recv_hook: bool, outs=None):
        n = len(self.ranks)
        stream = torch.cuda.current_stream().cuda_stream
        args = (L.LLCombineArgs * n)()
        res, keep = [], []
        for i in range(n):
            src_info, layout_range, Tm, H, E, route, comb_slot, count, k, use_proxy = handles[i]
            x = xs[i]
            if x.dtype != torch.bfloat16 or x.dim() != 3 or x.shape[2] != H:
                raise ConfigError("low_latency_combine expects bf16 x [num_local_experts, R*Tmax, hidden]")
            x = x.contiguous()
            topk_idx = topk_idxs[i].contiguous()
            w = topk_weights_list[i].to(torch.float32).contiguous()
            T = comb_slot.shape[0]
            if topk_idx.shape != comb_slot.shape or w.shape != comb_slot.shape:
                raise ProtocolViolation("topk_idx / topk_weights do not match the dispatch handle")
            out = outs[i] if outs is not None and outs[i] is not None else torch.empty(
                (T, H), dtype=torch.bfloat16, device=x.device)
            a = args[i]
            a.x, a.topk_idx, a.topk_weights = ptr(x), ptr(topk_idx), ptr(w)
            a.packed_recv_count, a.packed_recv_layout_range = ptr(count), ptr(layout_range)
            a.recv_route, a.comb_slot = ptr(route), ptr(comb_slot)
            a.num_tokens, a.num_topk, a.hidden, a.num_experts, a.max_tokens = T, k, H, E, Tm
            a.combined_x = ptr(out)
            a.phases = 1 if return_recv_hook else 3
            a.use_proxy = int(use_proxy)
            keep.append((x, topk_idx, w))
            res.append(out)
        self._launch("ll_combine", lambda: lib.epb_ll_combine(self._ctxs, n, args, _device_sms(), stream))
        hook = None
        if return_recv_hook:
            def hook(args=args, keep=keep):
                for i in range(n):
                    args[i].phases = 2
                check(lib.epb_ll_combine(self._ctxs, n, args, _device_sms(), torch.cuda.current_stream().cuda_stream))
        return res, hook

    def check_device_error(self) -> None:
        for rk in self.ranks:
            detail = C.c_int64()
            code = lib.epb_device_error(rk.ctx, C.byref(detail))
            if code:
                lib.epb_clear_device_error(rk.ctx)
                from .errors import raise_for
                raise_for(code, f"rank {rk.rank}: device reported error {code} (detail {detail.value:#x})")


def _event(async_finish: bool) -> EventOverlap:
    if not async_finish:
        return EventOverlap(None)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream())
    return EventOverlap(ev)


def _wait(previous_event: Optional[EventOverlap]) -> None:
    if previous_event is not None:
        previous_event.current_stream_wait()


class Buffer:
    """DeepEP-compatible communication buffer for one EP rank (one process per GPU)."""

    num_sms: int = 0  # 0 = every SM of the device

    def __init__(self, group=None, num_nvl_bytes: int = 0, num_rdma_bytes: int = 0, low_latency_mode: bool = False,
                 num_qps_per_rank: int = 24, allow_nvlink_for_low_latency_mode: bool = True,
                 allow_mnnvl: bool = False, explicitly_destroy: bool = False, *, num_recv_slots: int = 3,
                 fifo_channels: int = 8, fifo_capacity: int = 1024, proxy_threads: int = 4,
                 ll_transport: str = "nvlink"):
        import torch.distributed as dist
        if group is not None and dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
        if ll_transport not in ("nvlink", "proxy"):
            raise ConfigError("ll_transport must be 'nvlink' or 'proxy'")
        self.rank, self.group_size, self.group = rank, world, group
        self.low_latency_mode = low_latency_mode
        self.ll_transport = ll_transport
        self.num_nvl_bytes, self.num_rdma_bytes = int(num_nvl_bytes), int(num_rdma_bytes)
        ll_bytes = self.num_rdma_bytes if low_latency_mode else 0
        self._rank = _Rank(rank, world, max(self.num_nvl_bytes, 1 << 20), ll_bytes, num_recv_slots,
                           fifo_channels, fifo_capacity, proxy_threads)
        if world > 1:
            h = (C.c_char * L.IPC_HANDLE_BYTES)()
            check(lib.epb_ipc_handle(self._rank.ctx, h))
            handles: list = [None] * world
            dist.all_gather_object(handles, bytes(h), group=group)
            blob = b"".join(handles)
            check(lib.epb_open_peers(self._rank.ctx, blob))
            torch.cuda.synchronize()
            dist.barrier(group=group)
        else:
            check(lib.epb_link_local(_ctx_array([self._rank]), 1))
        if ll_transport == "proxy":
            check(lib.epb_proxy_start(self._rank.ctx))
            self._rank.proxy_running = True
        self._g = _Group([self._rank])
        self._destroyed = False

    # -- DeepEP helpers -------------------------------------------------------
    @staticmethod
    def set_num_sms(new_num_sms: int) -> None:
        Buffer.num_sms = int(new_num_sms)

    @staticmethod
    def get_dispatch_config(num_ranks: int) -> Config:
        return Config(Buffer.num_sms or None)

    @staticmethod
    def get_combine_config(num_ranks: int) -> Config:
        return Config(Buffer.num_sms or None)

    @staticmethod
    def get_low_latency_rdma_size_hint(num_max_dispatch_tokens_per_rank: int, hidden: int, num_ranks: int,
                                       num_experts: int, num_topk: Optional[int] = None) -> int:
        k = num_topk if num_topk is not None else num_experts // num_ranks
        lay = L.LLLayout()
        check(lib.epb_ll_layout(num_ranks, num_max_dispatch_tokens_per_rank, hidden, min(k, 32), num_experts, 1,
                                C.byref(lay)))
        return int(lay.bytes_needed)

    def get_local_buffer_tensor(self, dtype: torch.dtype = torch.uint8, size=None, offset: int = 0) -> torch.Tensor:
        mem = torch.as_tensor(_SlotMemory(self._rank.base, self._rank.region_bytes, None), device=self._rank.device)
        t = mem[offset:].view(dtype)
        return t if size is None else t[: int(torch.Size(size).numel())].view(size)

    def get_comm_stream(self) -> torch.cuda.Stream:
        return torch.cuda.current_stream()

    def destroy(self) -> None:
        if not self._destroyed:
            torch.cuda.synchronize()
            self._rank.destroy()
            self._destroyed = True

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def _config(self, config):
        return config if config is not None else Config(Buffer.num_sms or None)

    # -- layout -----------------------------------------------------------------
    def get_dispatch_layout(self, topk_idx: torch.Tensor, num_experts: int,
                            previous_event: Optional[EventOverlap] = None, async_finish: bool = False,
                            allocate_on_comm_stream: bool = False):
        _wait(previous_event)
        per_rank, per_rdma, per_expert, in_rank = self._g.get_dispatch_layout([topk_idx], num_experts)[0]
        return per_rank, per_rdma, per_expert, in_rank, _event(async_finish)

    # -- normal mode --------------------------------------------------------------
    def dispatch(self, x: Union[torch.Tensor, Tuple[torch.Tensor, torch.Tensor]], handle: Optional[tuple] = None,
                 num_tokens_per_rank: Optional[torch.Tensor] = None,
                 num_tokens_per_rdma_rank: Optional[torch.Tensor] = None,
                 is_token_in_rank: Optional[torch.Tensor] = None,
                 num_tokens_per_expert: Optional[torch.Tensor] = None, topk_idx: Optional[torch.Tensor] = None,
                 topk_weights: Optional[torch.Tensor] = None, expert_alignment: int = 1,
                 num_worst_tokens: int = 0, config: Optional[Config] = None,
                 previous_event: Optional[EventOverlap] = None, async_finish: bool = False,
                 allocate_on_comm_stream: bool = False):
        _wait(previous_event)
        (recv_x, recv_topk_idx, recv_topk_w, per_expert_list, new_handle), = self._g.dispatch(
            [x], [handle], [is_token_in_rank], [num_tokens_per_expert], [topk_idx], [topk_weights],
            expert_alignment, self._config(config))
        ev = _event(async_finish)
        if handle is not None:
            return recv_x, None, None, None, None, ev
        return recv_x, recv_topk_idx, recv_topk_w, per_expert_list, new_handle, ev

    def combine(self, x: torch.Tensor, handle: tuple, topk_weights: Optional[torch.Tensor] = None,
                bias=None, config: Optional[Config] = None, previous_event: Optional[EventOverlap] = None,
                async_finish: bool = False, allocate_on_comm_stream: bool = False):
        if bias is not None:
            raise UnsupportedOperation("combine bias is not supported")
        _wait(previous_event)
        (out, out_w), = self._g.combine([x], [handle], [topk_weights], self._config(config))
        return out, out_w, _event(async_finish)

    # -- low-latency mode -----------------------------------------------------------
    def low_latency_dispatch(self, x: torch.Tensor, topk_idx: torch.Tensor, num_max_dispatch_tokens_per_rank: int,
                             num_experts: int, cumulative_local_expert_recv_stats=None, use_fp8: bool = True,
                             round_scale: bool = False, use_ue8m0: bool = False, async_finish: bool = False,
                             return_recv_hook: bool = False):
        if not self.low_latency_mode:
            raise ConfigError("Buffer was not created with low_latency_mode=True")
        if use_ue8m0:
            raise UnsupportedOperation("UE8M0-packed scales are not supported; use round_scale=True for pow2 scales")
        res, hook = self._g.ll_dispatch(
            [x], [topk_idx], num_max_dispatch_tokens_per_rank, num_experts, use_fp8, round_scale, return_recv_hook,
            self.ll_transport == "proxy")
        recv, count, handle = res[0]
        if cumulative_local_expert_recv_stats is not None:
            cumulative_local_expert_recv_stats.add_(count)
        return recv, count, handle, _event(async_finish), hook

    def low_latency_combine(self, x: torch.Tensor, topk_idx: torch.Tensor, topk_weights: torch.Tensor,
                            handle: tuple, use_logfmt: bool = False, zero_copy: bool = False,
                            async_finish: bool = False, return_recv_hook: bool = False,
                            out: Optional[torch.Tensor] = None):
        if use_logfmt:
            raise UnsupportedOperation("LogFMT combine is not supported")
        (combined,), hook = self._g.ll_combine([x], [topk_idx], [topk_weights], [handle], return_recv_hook,
                                               [out])
        return combined, _event(async_finish), hook

    def clean_low_latency_buffer(self, num_max_dispatch_tokens_per_rank: int, hidden: int, num_experts: int) -> None:
        """Epoch-stamped flags never need clearing; kept for API compatibility."""
        return None

    def get_next_low_latency_combine_buffer(self, handle):
        raise UnsupportedOperation("zero-copy LL combine buffers are not exposed")


class LocalGroup:
    """R ranks in one process on one GPU (single-GPU multi-rank emulation).

    Methods take and return per-rank lists.  Every phase is one kernel launch
    over all ranks (cooperative where blocks wait on each other)."""

    def __init__(self, world: int, num_nvl_bytes: int, num_rdma_bytes: int = 0, *, num_recv_slots: int = 3,
                 fifo_channels: int = 0, fifo_capacity: int = 1024, proxy_threads: int = 1,
                 ll_transport: str = "nvlink"):
        if world < 1 or world > L.MAX_LOCAL:
            raise ConfigError("LocalGroup world must be in [1, 8]")
        self.ranks = [_Rank(r, world, num_nvl_bytes, num_rdma_bytes, num_recv_slots, fifo_channels, fifo_capacity,
                            proxy_threads) for r in range(world)]
        check(lib.epb_link_local(_ctx_array(self.ranks), world))
        self.ll_transport = ll_transport
        if ll_transport == "proxy":
            for rk in self.ranks:
                check(lib.epb_proxy_start(rk.ctx))
        self.world = world
        self._g = _Group(self.ranks)

    def get_dispatch_layout(self, topk_idx_list, num_experts):
        return self._g.get_dispatch_layout(topk_idx_list, num_experts)

    def dispatch(self, xs, is_token_in_ranks=None, num_tokens_per_experts=None, topk_idxs=None,
                 topk_weights_list=None, handles=None, expert_alignment=1, config=None):
        n = self.world
        handles = handles or [None] * n
        none = [None] * n
        return self._g.dispatch(xs, handles, is_token_in_ranks or none, num_tokens_per_experts or none,
                                topk_idxs or none, topk_weights_list or none, expert_alignment, config)

    def combine(self, xs, handles, topk_weights_list=None, config=None):
        return self._g.combine(xs, handles, topk_weights_list, config)

    def low_latency_dispatch(self, xs, topk_idxs, num_max_dispatch_tokens_per_rank, num_experts, use_fp8=True,
                             round_scale=False, return_recv_hook=False):
        return self._g.ll_dispatch(xs, topk_idxs, num_max_dispatch_tokens_per_rank, num_experts, use_fp8,
                                   round_scale, return_recv_hook, self.ll_transport == "proxy")

    def low_latency_combine(self, xs, topk_idxs, topk_weights_list, handles, return_recv_hook=False):
        return self._g.ll_combine(xs, topk_idxs, topk_weights_list, handles, return_recv_hook)

    def check_device_error(self):
        self._g.check_device_error()

    def destroy(self):
        torch.cuda.synchronize()
        for rk in self.ranks:
            rk.destroy()

    def __del__(self):
        try:
            for rk in self.ranks:
                rk.destroy()
        except Exception:
            pass
