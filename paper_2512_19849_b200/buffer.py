"""DeepEP-compatible ``Buffer`` for the B200 EP dispatch/combine path.

The paper claims drop-in compatibility with DeepEP's Python API
(PAPER.md:98); that API is not vendored in the reference, so the
signatures below follow DeepEP's public ``deep_ep.Buffer``.
Every data-path method goes through the C ABI (include/epb.h); the per-call
host work (shape checks, output allocation, argument structs, slot leases) runs
in the C++ runtime ``_epb_ext`` (csrc/ext/epb_ext.cpp), a client of that ABI:

* ``Buffer.__init__``        -> epb_create + CUDA-IPC handle all-gather + epb_open_peers
* ``get_dispatch_layout``    -> epb_get_dispatch_layout        (SPEC.md:416-424 plan_dedup)
* ``dispatch``               -> epb_dispatch + epb_wait_notify
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

import contextlib
import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple, Union

import torch

from . import _lib as L
from . import chunked
from ._lib import check, lib, raw_stream
from .errors import ConfigError, UnsupportedOperation, raise_for

from . import _epb_ext as X  # noqa: E402  (needs libepb200.so loaded by _lib)

_DEFAULT_TIMEOUT_S = float(os.environ.get("EPB_TIMEOUT_S", "30"))
_SMS_CACHE: dict = {}


def _device_sms() -> int:
    dev = torch._C._cuda_getDevice() if torch.cuda.is_available() else -1
    n = _SMS_CACHE.get(dev)
    if n is None:
        n = lib.epb_num_sms()
        n = n if n > 0 else 148
        _SMS_CACHE[dev] = n
    return n


@contextlib.contextmanager
def profiling(out: list):
    """Record (kernel-call name, device ms) for every launch inside the block."""
    X.set_profiling(True)
    try:
        yield out
    finally:
        X.set_profiling(False)
        out.extend(X.collect_profile())


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


def nvl_bytes_hint(num_tokens: int, hidden: int, num_ranks: int, num_topk: int = 8, num_slots: int = 3,
                   ht_proxy: bool = False) -> int:
    """Arena bytes so that the worst case (every token to every rank) fits:
    ``num_slots`` receive slots + 2 combine staging buffers of R*T rows (+ the
    send-staging slot of the proxy transport)."""
    rows = num_ranks * num_tokens
    per_row = 2 * hidden + 4 * (hidden // 128) + 12 * num_topk + 4
    comb_row = 2 * hidden + 4 * num_topk
    slots = num_slots + (1 if ht_proxy else 0)
    return rows * (slots * per_row + 2 * comb_row) + 256 * (6 * slots + 6) + (1 << 20)


def ring_nvl_bytes(hidden: int, num_ranks: int, num_topk: int = 8, lanes: int = 74, ring_tokens: int = 64) -> int:
    """Arena bytes for the chunked-ring transport (ht_transport="ring"): one
    dispatch ring and one combine ring of `ring_tokens` slots per (peer, lane)
    (csrc/chunked.cu ring_geometry) — independent of the token count."""
    def up(x, a):
        return (x + a - 1) // a * a
    S = hidden // 128
    o_sc = up(2 * hidden, 16)
    o_ti = up(o_sc + 4 * S, 8)
    disp = up(o_ti + 12 * num_topk + 12, 16)  # ... | src idx | receive row | canary
    comb = up(2 * hidden + 4 * num_topk + 4, 16)  # row | weights | canary
    return num_ranks * lanes * ring_tokens * (disp + comb)


def default_proxy_threads() -> int:
    """CPU proxy threads per rank when the caller does not choose: the paper's 4
     when the host has the cores, else what this rank's share of
    the cores leaves after its main thread (the threads spin while work is in
    flight, so oversubscribing cores stalls them for scheduler time slices)."""
    if os.environ.get("EPB_PROXY_THREADS"):
        return max(1, int(os.environ["EPB_PROXY_THREADS"]))
    cores = len(os.sched_getaffinity(0))
    ranks_here = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    return max(1, min(4, cores // max(1, ranks_here) - 1))


_HT_CODES = {"nvlink": L.HT_NVLINK, "proxy": L.HT_PROXY, "ring": L.HT_RING}


class _SlotMemory:
    """``__cuda_array_interface__`` over raw device memory (debug views)."""

    def __init__(self, addr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (addr, False), "version": 3,
                                         "strides": None, "stream": None}


class _Rank:
    """Native state of one EP rank: the epb_t* plus the C++ runtime's rank
    object (receive-slot pool, cached arena geometry)."""

    def __init__(self, rank: int, world: int, nvl_bytes: int, ll_bytes: int, num_recv_slots: int,
                 fifo_channels: int, fifo_capacity: int, proxy_threads: int, ht_transport: str = "nvlink"):
        self.rank, self.world = rank, world
        self.device = torch.device("cuda", torch.cuda.current_device())
        cfg = L.Config(nvl_bytes, ll_bytes, num_recv_slots, fifo_channels, fifo_capacity, proxy_threads,
                       _HT_CODES[ht_transport])
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
        self.native = X.Rank(ctx.value, rank, world, self.num_slots, self.base, self.device.index)
        self.proxy_running = False

    def num_free_slots(self) -> int:
        return self.native.num_free_slots()

    def destroy(self) -> None:
        if self.ctx:
            lib.epb_destroy(self.ctx)
            self.ctx = None


def _ctx_array(ranks: Sequence[_Rank]):
    return (C.c_void_p * len(ranks))(*[r.ctx.value for r in ranks])


def _split_x(x):
    if isinstance(x, tuple):
        return x[0], x[1]
    return x, None


class _Group:
    """List-based implementation shared by Buffer (1 rank) and LocalGroup (R ranks)."""

    def __init__(self, ranks: List[_Rank], ht_transport: str = "nvlink", ring_lanes: int = 0):
        self.ranks = ranks
        self.native = [r.native for r in ranks]
        self.world = ranks[0].world
        self.timeout_s = _DEFAULT_TIMEOUT_S
        self.ring = ht_transport == "ring"
        self.ring_lanes = ring_lanes

    def get_dispatch_layout(self, topk_idx_list: Sequence[torch.Tensor], num_experts: int):
        out = []
        for topk_idx in topk_idx_list:
            per_rank, per_expert, in_rank = X.layout(topk_idx, num_experts, self.world)
            out.append((per_rank, None, per_expert, in_rank))
        return out

    def dispatch(self, xs, handles, is_token_in_ranks, num_tokens_per_experts, topk_idxs, topk_weights_list,
                 expert_alignment: int, config: Optional[Config], num_worst_tokens: int = 0):
        n = len(self.ranks)
        cfg = config or Config()
        # one block per channel; all blocks of all local ranks must be co-resident
        channels = max(1, min(cfg.resolved_sms(), _device_sms() // n))
        xd, xsc = zip(*[_split_x(x) for x in xs])
        if self.ring:  # bounded chunked rings (chunked.py / csrc/chunked.cu)
            if handles[0] is not None:
                in_ranks, none = [h[4] for h in handles], [None] * n
                return chunked.ring_dispatch(self.ranks, xd, xsc, in_ranks, none, none, none, expert_alignment,
                                             channels, self.timeout_s, self.ring_lanes)
            return chunked.ring_dispatch(self.ranks, xd, xsc, is_token_in_ranks, num_tokens_per_experts, topk_idxs,
                                         topk_weights_list, expert_alignment, channels, self.timeout_s,
                                         self.ring_lanes)
        if handles[0] is not None:  # cached layout: the handle carries is_token_in_rank
            in_ranks = [h[4] for h in handles]
            none = [None] * n
            return X.dispatch(self.native, list(xd), list(xsc), in_ranks, none, none, none, expert_alignment,
                              channels, self.timeout_s, int(num_worst_tokens))
        for ir in is_token_in_ranks:
            if ir is None:
                raise ConfigError("is_token_in_rank is required without a handle")
        return X.dispatch(self.native, list(xd), list(xsc), list(is_token_in_ranks), list(num_tokens_per_experts),
                          list(topk_idxs), list(topk_weights_list), expert_alignment, channels, self.timeout_s,
                          int(num_worst_tokens))

    def combine(self, xs, handles, topk_weights_list, config: Optional[Config]):
        cfg = config or Config()
        ws = list(topk_weights_list) if topk_weights_list is not None else [None] * len(xs)
        if self.ring:
            return chunked.ring_combine(self.ranks, list(xs), list(handles), ws, self.ring_lanes)
        return X.combine(self.native, list(xs), list(handles), ws, cfg.resolved_sms())

    def ll_dispatch(self, xs, topk_idxs, num_max_dispatch_tokens_per_rank: int, num_experts: int, use_fp8: bool,
                    round_scale: bool, return_recv_hook: bool, use_proxy: bool):
        res, hook = X.ll_dispatch(self.native, list(xs), list(topk_idxs), int(num_max_dispatch_tokens_per_rank),
                                  int(num_experts), bool(use_fp8), bool(round_scale), bool(return_recv_hook),
                                  bool(use_proxy), _device_sms())
        return list(res), hook

    def ll_combine(self, xs, topk_idxs, topk_weights_list, handles, return_recv_hook: bool, outs=None):
        outs = list(outs) if outs is not None else [None] * len(xs)
        res, hook = X.ll_combine(self.native, list(xs), list(topk_idxs), list(topk_weights_list), list(handles),
                                 bool(return_recv_hook), outs, _device_sms())
        return list(res), hook

    def check_device_error(self) -> None:
        for rk in self.ranks:
            detail = C.c_int64()
            code = lib.epb_device_error(rk.ctx, C.byref(detail))
            if code:
                lib.epb_clear_device_error(rk.ctx)
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


def _tensors(obj, out=None):
    out = [] if out is None else out
    if isinstance(obj, torch.Tensor):
        out.append(obj)
    elif isinstance(obj, (tuple, list)):
        for o in obj:
            _tensors(o, out)
    return out


def _record(t: torch.Tensor, stream) -> None:
    try:  # zero-copy views of the symmetric region are not caching-allocator memory
        t.record_stream(stream)
    except RuntimeError:
        pass


class _CommStream:
    """DeepEP's stream discipline for one op (deep_ep Buffer: previous_event /
    async_finish / allocate_on_comm_stream).  The op runs on the Buffer's comm
    stream after ``previous_event`` (or after the current compute stream); with
    async_finish the caller gets an EventOverlap on the comm stream and the
    tensors involved are recorded on it, otherwise the compute stream waits
    for the comm stream before the call returns.  With none of the three
    options the op runs on the compute stream directly (the same ordering,
    without the stream hops)."""

    def __init__(self, buf: "Buffer", previous_event, async_finish: bool, allocate_on_comm_stream: bool, inputs=()):
        self.active = previous_event is not None or async_finish or allocate_on_comm_stream
        self.buf, self.prev, self.async_finish, self.inputs = buf, previous_event, async_finish, inputs

    def __enter__(self):
        if not self.active:
            return self
        self.compute = torch.cuda.current_stream()
        comm = self.buf._comm_stream()
        if self.prev is not None and self.prev.event is not None:
            comm.wait_event(self.prev.event)
        else:
            comm.wait_stream(self.compute)
        self.ctx = torch.cuda.stream(comm)
        self.ctx.__enter__()
        return self

    def finish(self, result) -> EventOverlap:
        if not self.active:
            return EventOverlap(None)
        self.ctx.__exit__(None, None, None)
        comm = self.buf._comm_stream()
        ts = _tensors(result) + _tensors(self.inputs)
        if self.async_finish:
            ev = torch.cuda.Event()
            ev.record(comm)
            for t in ts:  # caching-allocator safety: in use on both streams
                _record(t, comm)
                _record(t, self.compute)
            return EventOverlap(ev, ts)
        self.compute.wait_stream(comm)
        for t in _tensors(result):
            _record(t, self.compute)
        return EventOverlap(None)

    def __exit__(self, exc_type, exc, tb):
        if exc_type is not None and self.active:
            self.ctx.__exit__(exc_type, exc, tb)
        return False


class Buffer:
    """DeepEP-compatible communication buffer for one EP rank (one process per GPU)."""

    num_sms: int = 0  # 0 = every SM of the device

    def __init__(self, group=None, num_nvl_bytes: int = 0, num_rdma_bytes: int = 0, low_latency_mode: bool = False,
                 num_qps_per_rank: int = 24, allow_nvlink_for_low_latency_mode: bool = True,
                 allow_mnnvl: bool = False, explicitly_destroy: bool = False, *, num_recv_slots: int = 3,
                 fifo_channels: int = 8, fifo_capacity: int = 1024, proxy_threads: int = 0,
                 ll_transport: str = "nvlink", ht_transport: str = "nvlink", ring_lanes: int = 0):
        import torch.distributed as dist
        if group is not None and dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
        if ll_transport not in ("nvlink", "proxy") or ht_transport not in ("nvlink", "proxy", "ring"):
            raise ConfigError("ll_transport must be 'nvlink' or 'proxy'; ht_transport 'nvlink', 'proxy' or 'ring'")
        if ht_transport == "proxy" and fifo_channels <= 0:
            raise ConfigError("ht_transport='proxy' needs fifo_channels > 0")
        self.ht_transport = ht_transport
        self.rank, self.group_size, self.group = rank, world, group
        self.low_latency_mode = low_latency_mode
        self.ll_transport = ll_transport
        self.num_nvl_bytes, self.num_rdma_bytes = int(num_nvl_bytes), int(num_rdma_bytes)
        ll_bytes = self.num_rdma_bytes if low_latency_mode else 0
        self._rank = _Rank(rank, world, max(self.num_nvl_bytes, 1 << 20), ll_bytes, num_recv_slots,
                           fifo_channels, fifo_capacity, proxy_threads or default_proxy_threads(), ht_transport=ht_transport)
        if world > 1:
            h = (C.c_char * L.IPC_HANDLE_BYTES)()
            check(lib.epb_ipc_handle(self._rank.ctx, h))
            handles = exchange_handles(bytes(h), world, group)
            check(lib.epb_open_peers(self._rank.ctx, b"".join(handles)))
            torch.cuda.synchronize()
            dist.barrier(group=group)
        else:
            check(lib.epb_link_local(_ctx_array([self._rank]), 1))
        if ll_transport == "proxy" or ht_transport == "proxy":
            self.start_proxy()
        self._g = _Group([self._rank], ht_transport, ring_lanes)
        self._native = self._rank.native
        self._sms_key, self._sms_val = None, 0
        self._comm = None
        self._ll_comb_bufs = {}
        self._destroyed = False

    def start_proxy(self) -> None:
        """Start the CPU proxy threads that drain this rank's GPU->CPU FIFOs."""
        if not self._rank.proxy_running:
            check(lib.epb_proxy_start(self._rank.ctx))
            self._rank.proxy_running = True

    def proxy_barrier(self, channel: int = 0, same_rail: bool = False) -> None:
        """Stream-ordered all-peer barrier through the GPU->CPU FIFO: a kernel
        pushes a Barrier TransferCmd on `channel` and waits on its completion,
        which the proxy grants once every rank's proxy has entered
        (PAPER.md:313-315)."""
        self.start_proxy()
        check(lib.epb_proxy_barrier(self._rank.ctx, int(channel), int(bool(same_rail)), raw_stream()))

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
        mem = torch.as_tensor(_SlotMemory(self._rank.base, self._rank.region_bytes), device=self._rank.device)
        t = mem[offset:].view(dtype)
        return t if size is None else t[: int(torch.Size(size).numel())].view(size)

    def _comm_stream(self) -> torch.cuda.Stream:
        if self._comm is None:
            self._comm = torch.cuda.Stream(device=self._rank.device)
        return self._comm

    def get_comm_stream(self) -> torch.cuda.Stream:
        """The stream ops run on when async_finish / previous_event /
        allocate_on_comm_stream are given (DeepEP Buffer.get_comm_stream)."""
        return self._comm_stream()

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

    def _sms(self, config) -> int:
        """SMs (= dispatch channels) for this call; one process per GPU."""
        if config is not None:
            return max(1, min(config.resolved_sms(), _device_sms()))
        key = Buffer.num_sms
        if self._sms_key != key:
            self._sms_key, self._sms_val = key, max(1, min(Config(key or None).resolved_sms(), _device_sms()))
        return self._sms_val

    # -- layout -----------------------------------------------------------------
    def get_dispatch_layout(self, topk_idx: torch.Tensor, num_experts: int,
                            previous_event: Optional[EventOverlap] = None, async_finish: bool = False,
                            allocate_on_comm_stream: bool = False):
        with _CommStream(self, previous_event, async_finish, allocate_on_comm_stream, (topk_idx,)) as cs:
            per_rank, per_expert, in_rank = X.layout(topk_idx, num_experts, self.group_size)
            ev = cs.finish((per_rank, per_expert, in_rank))
        return per_rank, None, per_expert, in_rank, ev

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
        with _CommStream(self, previous_event, async_finish, allocate_on_comm_stream,
                         (x, topk_idx, topk_weights, is_token_in_rank)) as cs:
            r = self._dispatch(x, handle, is_token_in_rank, num_tokens_per_expert, topk_idx, topk_weights,
                               expert_alignment, num_worst_tokens, config)
            ev = cs.finish((r[0], r[1], r[2], r[4]))
        return r[0], r[1], r[2], r[3], r[4], ev

    def _dispatch(self, x, handle, is_token_in_rank, num_tokens_per_expert, topk_idx, topk_weights, expert_alignment,
                  num_worst_tokens, config):
        xd, xs = (x[0], x[1]) if isinstance(x, tuple) else (x, None)
        if self.ht_transport == "ring":
            if handle is None and is_token_in_rank is None:
                raise ConfigError("is_token_in_rank is required without a handle")
            (r,) = self._g.dispatch([x], [handle], [is_token_in_rank], [num_tokens_per_expert], [topk_idx],
                                    [topk_weights], expert_alignment, self._config(config))
            if handle is not None:
                return r[0], None, None, None, None
            return r[0], r[1], r[2], r[3], r[4]
        if num_worst_tokens and self.ht_transport != "nvlink":
            raise UnsupportedOperation("num_worst_tokens needs ht_transport='nvlink' (the proxy and ring transports "
                                       "size their outputs from a host sync)")
        if handle is not None:  # cached layout: the handle carries is_token_in_rank
            r = X.dispatch1(self._native, xd, xs, handle[4], None, None, None, expert_alignment, self._sms(config),
                            self._g.timeout_s, int(num_worst_tokens))
            return r[0], None, None, None, None
        if is_token_in_rank is None:
            raise ConfigError("is_token_in_rank is required without a handle")
        r = X.dispatch1(self._native, xd, xs, is_token_in_rank, num_tokens_per_expert, topk_idx, topk_weights,
                        expert_alignment, self._sms(config), self._g.timeout_s, int(num_worst_tokens))
        return r[0], r[1], r[2], r[3], r[4]

    def combine(self, x: torch.Tensor, handle: tuple, topk_weights: Optional[torch.Tensor] = None,
                bias=None, config: Optional[Config] = None, previous_event: Optional[EventOverlap] = None,
                async_finish: bool = False, allocate_on_comm_stream: bool = False):
        if bias is not None:
            raise UnsupportedOperation("combine bias is not supported")
        with _CommStream(self, previous_event, async_finish, allocate_on_comm_stream, (x, topk_weights)) as cs:
            if self.ht_transport == "ring":
                ((out, out_w),) = self._g.combine([x], [handle], [topk_weights], config)
            else:
                out, out_w = X.combine1(self._native, x, handle, topk_weights, self._sms(config))
            ev = cs.finish((out, out_w))
        return out, out_w, ev

    # -- low-latency mode -----------------------------------------------------------
    def low_latency_dispatch(self, x: torch.Tensor, topk_idx: torch.Tensor, num_max_dispatch_tokens_per_rank: int,
                             num_experts: int, cumulative_local_expert_recv_stats=None, use_fp8: bool = True,
                             round_scale: bool = False, use_ue8m0: bool = False, async_finish: bool = False,
                             return_recv_hook: bool = False):
        if not self.low_latency_mode:
            raise ConfigError("Buffer was not created with low_latency_mode=True")
        if use_ue8m0:
            raise UnsupportedOperation("UE8M0-packed scales are not supported; use round_scale=True for pow2 scales")
        with _CommStream(self, None, async_finish, False, (x, topk_idx)) as cs:
            res, hook = self._g.ll_dispatch([x], [topk_idx], num_max_dispatch_tokens_per_rank, num_experts, use_fp8,
                                            round_scale, return_recv_hook, self.ll_transport == "proxy")
            recv, count, handle = res[0]
            if cumulative_local_expert_recv_stats is not None:
                cumulative_local_expert_recv_stats.add_(count)
            ev = cs.finish((recv, count))
        return recv, count, handle, ev, hook

    def low_latency_combine(self, x: torch.Tensor, topk_idx: torch.Tensor, topk_weights: torch.Tensor,
                            handle: tuple, use_logfmt: bool = False, zero_copy: bool = False,
                            async_finish: bool = False, return_recv_hook: bool = False,
                            out: Optional[torch.Tensor] = None):
        if use_logfmt:
            raise UnsupportedOperation("LogFMT combine is not supported")
        # zero_copy: x may be the tensor get_next_low_latency_combine_buffer returned;
        # the kernel reads expert outputs wherever they live, so both paths are the same
        with _CommStream(self, None, async_finish, False, (x, topk_idx, topk_weights)) as cs:
            (combined,), hook = self._g.ll_combine([x], [topk_idx], [topk_weights], [handle], return_recv_hook,
                                                   [out])
            ev = cs.finish((combined,))
        return combined, ev, hook

    def clean_low_latency_buffer(self, num_max_dispatch_tokens_per_rank: int, hidden: int, num_experts: int) -> None:
        """Epoch-stamped flags never need clearing; kept for API compatibility."""
        return None

    def get_next_low_latency_combine_buffer(self, handle):
        """DeepEP zero-copy combine: a [num_local_experts, R*Tmax, hidden] bf16
        buffer the experts can write into, then passed to
        low_latency_combine(..., zero_copy=True).  Two buffers alternate per
        call, like DeepEP's double-buffered low-latency region."""
        Tm, H, E = int(handle[2]), int(handle[3]), int(handle[4])
        key = (Tm, H, E)
        pair = self._ll_comb_bufs.get(key)
        if pair is None:
            shape = (E // self.group_size, self.group_size * Tm, H)
            pair = [[torch.empty(shape, dtype=torch.bfloat16, device=self._rank.device) for _ in range(2)], 0]
            self._ll_comb_bufs[key] = pair
        pair[1] ^= 1
        return pair[0][pair[1]]


def exchange_handles(my_handle: bytes, world: int, group=None) -> List[bytes]:
    """All-gather the ranks' CUDA-IPC handles (bootstrap only; the single use of
    torch.distributed in the library)."""
    import torch.distributed as dist
    handles: list = [None] * world
    dist.all_gather_object(handles, my_handle, group=group)
    for h in handles:
        if not isinstance(h, bytes) or len(h) != L.IPC_HANDLE_BYTES:
            raise ConfigError("malformed IPC handle from a peer")
    return handles


class LocalGroup:
    """R ranks in one process on one GPU (single-GPU multi-rank emulation).

    Methods take and return per-rank lists.  Every phase is one kernel launch
    over all ranks (cooperative where blocks wait on each other)."""

    def __init__(self, world: int, num_nvl_bytes: int, num_rdma_bytes: int = 0, *, num_recv_slots: int = 3,
                 fifo_channels: int = 0, fifo_capacity: int = 1024, proxy_threads: int = 1,
                 ll_transport: str = "nvlink", ht_transport: str = "nvlink", ring_lanes: int = 0):
        if world < 1 or world > L.MAX_LOCAL:
            raise ConfigError("LocalGroup world must be in [1, 8]")
        if ht_transport == "proxy" and fifo_channels <= 0:
            raise ConfigError("ht_transport='proxy' needs fifo_channels > 0")
        self.ranks = [_Rank(r, world, num_nvl_bytes, num_rdma_bytes, num_recv_slots, fifo_channels, fifo_capacity,
                            proxy_threads, ht_transport=ht_transport) for r in range(world)]
        check(lib.epb_link_local(_ctx_array(self.ranks), world))
        self.ll_transport = ll_transport
        self.ht_transport = ht_transport
        if ll_transport == "proxy" or ht_transport == "proxy":
            for rk in self.ranks:
                check(lib.epb_proxy_start(rk.ctx))
                rk.proxy_running = True
        self.world = world
        self._g = _Group(self.ranks, ht_transport, ring_lanes)

    def get_dispatch_layout(self, topk_idx_list, num_experts):
        return self._g.get_dispatch_layout(topk_idx_list, num_experts)

    def dispatch(self, xs, is_token_in_ranks=None, num_tokens_per_experts=None, topk_idxs=None,
                 topk_weights_list=None, handles=None, expert_alignment=1, config=None, num_worst_tokens=0):
        n = self.world
        handles = handles or [None] * n
        none = [None] * n
        return self._g.dispatch(xs, handles, is_token_in_ranks or none, num_tokens_per_experts or none,
                                topk_idxs or none, topk_weights_list or none, expert_alignment, config,
                                num_worst_tokens)

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
