"""ctypes binding of libepb200.so (the C ABI declared in include/epb.h).

The library is the product: there is no Python or CPU fallback.  If the .so is
missing or fails to load, importing this module raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import raise_for

LIB_PATH = Path(__file__).resolve().parent / "libepb200.so"

MAX_RANKS = 8
MAX_LOCAL = 8
MAX_CHANNELS = 256
MAX_LOCAL_EXPERTS = 1024
IPC_HANDLE_BYTES = 64

CTL_TAIL, CTL_HEAD, CTL_COMPLETED, CTL_FLAGS, CTL_SLOT0 = 0, 8, 16, 24, 32

HT_NVLINK, HT_PROXY, HT_RING = 0, 1, 2  # epb_config_t.ht_transport (EPB_HT_*)


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(no CPU fallback exists for the EP path)")
    return C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | C.RTLD_GLOBAL)


lib = _load()

vp = C.c_void_p
i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64
P64 = C.POINTER(C.c_int64)
PU64 = C.POINTER(C.c_uint64)
P32 = C.POINTER(C.c_int32)


class Config(C.Structure):
    _fields_ = [("nvl_bytes", C.c_size_t), ("ll_bytes", C.c_size_t), ("num_recv_slots", C.c_int),
                ("fifo_channels", C.c_int), ("fifo_capacity", C.c_int), ("proxy_threads", C.c_int),
                ("ht_transport", C.c_int)]


class RecvLayout(C.Structure):
    _fields_ = [("cap_rows", i64), ("slot_bytes", i64), ("off_x", i64), ("off_scales", i64),
                ("off_topk_idx", i64), ("off_topk_w", i64), ("off_src_idx", i64), ("comb_off", i64 * 2),
                ("comb_w_off", i64), ("slot0_off", i64), ("send_off", i64),
                ("comb_flag_off", i64)]


class DispatchArgs(C.Structure):
    _fields_ = [("x", vp), ("x_scales", vp), ("hidden", C.c_int), ("elem_bytes", C.c_int), ("num_scales", C.c_int),
                ("topk_idx", vp), ("topk_weights", vp), ("num_topk", C.c_int), ("is_token_in_rank", vp),
                ("num_tokens_per_expert", vp), ("num_tokens", C.c_int), ("num_experts", C.c_int),
                ("expert_alignment", C.c_int), ("recv_slot", C.c_int), ("rank_prefix_matrix", vp),
                ("channel_prefix_matrix", vp), ("recv_channel_prefix_matrix", vp), ("send_head", vp),
                ("num_worst_tokens", C.c_int)]


class CombineArgs(C.Structure):
    _fields_ = [("x", vp), ("topk_weights", vp), ("num_recv", C.c_int), ("hidden", C.c_int), ("num_topk", C.c_int),
                ("rank_prefix_matrix", vp), ("is_token_in_rank", vp), ("send_head", vp),
                ("channel_prefix_matrix", vp), ("recv_channel_prefix_matrix", vp), ("num_channels", C.c_int),
                ("num_tokens", C.c_int),
                ("combined_x", vp), ("combined_topk_weights", vp)]


class RingLayout(C.Structure):
    _fields_ = [("lanes", C.c_int), ("ring_tokens", C.c_int), ("disp_slot_bytes", i64), ("comb_slot_bytes", i64),
                ("disp_off", i64), ("comb_off", i64), ("bytes_needed", i64)]


class RingDispatchArgs(C.Structure):
    _fields_ = [("x", vp), ("x_scales", vp), ("hidden", C.c_int), ("elem_bytes", C.c_int), ("num_scales", C.c_int),
                ("topk_idx", vp), ("topk_weights", vp), ("num_topk", C.c_int), ("num_tokens", C.c_int),
                ("num_experts", C.c_int), ("rank_prefix_matrix", vp), ("recv_channel_prefix_matrix", vp),
                ("send_head", vp), ("num_channels", C.c_int), ("recv_x", vp), ("recv_x_scales", vp),
                ("recv_topk_idx", vp), ("recv_topk_weights", vp), ("recv_src_idx", vp), ("num_recv", C.c_int)]


class RingCombineArgs(C.Structure):
    _fields_ = [("x", vp), ("topk_weights", vp), ("num_recv", C.c_int), ("hidden", C.c_int), ("num_topk", C.c_int),
                ("rank_prefix_matrix", vp), ("recv_channel_prefix_matrix", vp), ("send_head", vp),
                ("num_channels", C.c_int), ("num_tokens", C.c_int), ("combined_x", vp),
                ("combined_topk_weights", vp)]


class LLLayout(C.Structure):
    _fields_ = [("rows_per_src", i64), ("disp_row_bytes", i64), ("comb_row_bytes", i64), ("bytes_needed", i64)]


class LLDispatchArgs(C.Structure):
    _fields_ = [("x", vp), ("topk_idx", vp), ("num_tokens", C.c_int), ("num_topk", C.c_int), ("hidden", C.c_int),
                ("num_experts", C.c_int), ("max_tokens", C.c_int), ("use_fp8", C.c_int), ("round_scale", C.c_int),
                ("packed_recv_x", vp), ("packed_recv_x_scales", vp), ("packed_recv_count", vp),
                ("packed_recv_src_info", vp), ("packed_recv_layout_range", vp), ("recv_route", vp),
                ("comb_slot", vp), ("phases", C.c_int), ("use_proxy", C.c_int)]


class LLCombineArgs(C.Structure):
    _fields_ = [("x", vp), ("topk_idx", vp), ("topk_weights", vp), ("packed_recv_count", vp),
                ("packed_recv_layout_range", vp), ("recv_route", vp), ("comb_slot", vp), ("num_tokens", C.c_int),
                ("num_topk", C.c_int), ("hidden", C.c_int), ("num_experts", C.c_int), ("max_tokens", C.c_int),
                ("combined_x", vp), ("phases", C.c_int), ("use_proxy", C.c_int)]


def _proto(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


CTXS = C.POINTER(vp)
c_int, c_double = C.c_int, C.c_double

_proto("epb_last_error", C.c_char_p)
_proto("epb_create", c_int, C.POINTER(vp), c_int, c_int, C.POINTER(Config))
_proto("epb_destroy", c_int, vp)
_proto("epb_ipc_handle", c_int, vp, vp)
_proto("epb_open_peers", c_int, vp, vp)
_proto("epb_link_local", c_int, CTXS, c_int)
_proto("epb_device_error", c_int, vp, P64)
_proto("epb_clear_device_error", c_int, vp)
_proto("epb_num_sms", c_int)
_proto("epb_region", c_int, vp, C.POINTER(vp), C.POINTER(C.c_size_t))
_proto("epb_trace", c_int, vp, P64)
_proto("epb_debug_stamp", c_int, vp, vp)
_proto("epb_debug_ht_sig_offset", i64)
_proto("epb_get_dispatch_layout", c_int, vp, c_int, c_int, c_int, c_int, vp, vp, vp, vp)
_proto("epb_recv_layout", c_int, vp, c_int, c_int, C.POINTER(RecvLayout))
_proto("epb_wait_notify", c_int, vp, P64, P32, c_int, c_double)
_proto("epb_dispatch", c_int, CTXS, c_int, C.POINTER(DispatchArgs), c_int, vp)
_proto("epb_combine", c_int, CTXS, c_int, C.POINTER(CombineArgs), c_int, vp)
_proto("epb_ring_layout", c_int, vp, c_int, c_int, c_int, c_int, C.POINTER(RingLayout))
_proto("epb_dispatch_notify", c_int, CTXS, c_int, C.POINTER(DispatchArgs), c_int, vp)
_proto("epb_ring_dispatch", c_int, CTXS, c_int, C.POINTER(RingDispatchArgs), c_int, vp)
_proto("epb_ring_combine", c_int, CTXS, c_int, C.POINTER(RingCombineArgs), c_int, vp)
_proto("epb_ll_layout", c_int, c_int, c_int, c_int, c_int, c_int, c_int, C.POINTER(LLLayout))
_proto("epb_ll_dispatch", c_int, CTXS, c_int, C.POINTER(LLDispatchArgs), c_int, vp)
_proto("epb_ll_combine", c_int, CTXS, c_int, C.POINTER(LLCombineArgs), c_int, vp)
_proto("epb_per_token_cast_to_fp8", c_int, vp, c_int, c_int, c_int, vp, vp, vp)
_proto("epb_cmd_pack", c_int, i64, i64, i64, i64, i64, i64, i64, PU64, PU64)
_proto("epb_cmd_pack_fields", c_int, P64, P64, P64, P64, P64, P64, P64, i64, PU64, PU64)
_proto("epb_cmd_unpack_fields", c_int, PU64, PU64, i64, P64, P64, P64, P64, P64, P64, P64)
_proto("epb_imm_encode_ll_batch", c_int, P64, P64, P64, i64, P64)
_proto("epb_imm_encode_ht_batch", c_int, P64, P64, P64, P64, i64, P64)
_proto("epb_ring_push_batch", i64, P64, i64, P64, P64, i64, i64, i64)
_proto("epb_ring_pop_batch", i64, P64, i64, P64, P64, i64, i64, i64)
_proto("epb_ring_poll", c_int, P64, i64, P64, P64)
_proto("epb_ring_mark_completed", c_int, P64, i64)
_proto("epb_ring_check_completion", c_int, P64, i64)
_proto("epb_ring_shutdown", c_int, P64)
_proto("epb_apply_deliveries", c_int,
       vp, i64, i64, P64, i64, i64, i64, i64, i64,  # regions .. n
       P64, P64, P64, P64, P64, P64, P64, P64, P64,  # t_del .. work_id
       P64, P32, P32, P32, i64, P64, P32, i64, i64,  # ll_counts .. wmax
       P64, P64, P64, P64, P64, P64, P64, P64, i64,  # eff_* .. eff_cap
       P64, i64, P64)
_proto("epb_fifo_ctl", c_int, vp, c_int, C.POINTER(P64), P64)
_proto("epb_proxy_start", c_int, vp)
_proto("epb_proxy_stop", c_int, vp)
_proto("epb_proxy_stats", c_int, vp, P64)
_proto("epb_fifo_device_bench", c_int, vp, i64, c_int, P64, vp)
_proto("epb_barrier_open", c_int, C.c_char_p, c_int, c_int, C.POINTER(vp))
_proto("epb_barrier_wait", c_int, vp, c_int, c_double)
_proto("epb_barrier_close", c_int, vp, c_int)
_proto("epb_proxy_barrier", c_int, vp, c_int, c_int, vp)
_proto("epb_proxy_drain", c_int, vp, c_int, i64, vp)
_proto("epb_arena_offset", i64)
_proto("epb_debug_ll_state", c_int, vp, P64)
_proto("epb_debug_drain_test", c_int, vp, c_int, c_int, c_int, i64, i64, i64, i64, vp, vp)
_proto("epb_proxy_trace", i64, vp, P64, i64)
_proto("epb_clock_calibrate", c_int, P64, P64)

# every symbol include/epb.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "epb_create", "epb_destroy", "epb_ipc_handle", "epb_open_peers", "epb_link_local", "epb_last_error",
    "epb_device_error", "epb_clear_device_error", "epb_num_sms", "epb_region", "epb_trace", "epb_debug_stamp", "epb_debug_ht_sig_offset", "epb_get_dispatch_layout",
    "epb_recv_layout", "epb_wait_notify", "epb_dispatch", "epb_combine", "epb_ring_layout", "epb_dispatch_notify",
    "epb_ring_dispatch", "epb_ring_combine", "epb_ll_layout",
    "epb_ll_dispatch", "epb_ll_combine", "epb_per_token_cast_to_fp8", "epb_cmd_pack", "epb_cmd_pack_fields",
    "epb_cmd_unpack_fields", "epb_imm_encode_ll_batch", "epb_imm_encode_ht_batch", "epb_ring_push_batch",
    "epb_ring_pop_batch", "epb_ring_poll", "epb_ring_mark_completed", "epb_ring_check_completion",
    "epb_ring_shutdown", "epb_apply_deliveries", "epb_fifo_ctl", "epb_proxy_start", "epb_proxy_stop",
    "epb_proxy_stats", "epb_fifo_device_bench", "epb_barrier_open", "epb_barrier_wait", "epb_barrier_close",
    "epb_proxy_barrier", "epb_proxy_drain", "epb_debug_drain_test", "epb_proxy_trace", "epb_clock_calibrate",
    "epb_arena_offset", "epb_debug_ll_state",
]


def raw_stream() -> int:
    """cudaStream_t of torch's current stream on the current device (the cheap
    path; torch.cuda.current_stream() costs ~10 us of Python per call)."""
    import torch
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def check(rc: int) -> None:
    """Raise the reference's exception class for a non-zero EPB code."""
    if rc != 0:
        raise_for(rc, lib.epb_last_error().decode(errors="replace"))


def ptr(t) -> int:
    """Device/host address of a torch tensor or numpy array (None -> 0)."""
    if t is None:
        return 0
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def nptr(a, ctype):
    """ctypes typed pointer into a contiguous numpy array."""
    return a.ctypes.data_as(C.POINTER(ctype))
