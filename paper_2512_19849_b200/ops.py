"""Standalone device ops of the path."""
from __future__ import annotations

import torch

from ._lib import check, lib, ptr, raw_stream
from .errors import ConfigError


def per_token_cast_to_fp8(x: torch.Tensor, round_scale: bool = False):
    """bf16 [T, H] -> (e4m3 [T, H], f32 scales [T, H/128]); the LL dispatch quantiser
    (ll.cu quant16; formula pinned in oracle/ep.py:fp8_quant)."""
    if x.dtype != torch.bfloat16 or x.dim() != 2 or x.shape[1] % 128:
        raise ConfigError("expected bf16 [T, H] with H % 128 == 0")
    x = x.contiguous()
    T, H = x.shape
    q = torch.empty((T, H), dtype=torch.float8_e4m3fn, device=x.device)
    s = torch.empty((T, H // 128), dtype=torch.float32, device=x.device)
    check(lib.epb_per_token_cast_to_fp8(ptr(x), T, H, int(round_scale), ptr(q), ptr(s),
                                        raw_stream()))
    return q, s


def get_dispatch_layout(topk_idx: torch.Tensor, num_experts: int, num_ranks: int):
    """topk_idx int64 [T, k] -> (num_tokens_per_rank i32 [R], num_tokens_per_expert i32 [E],
    is_token_in_rank bool [T, R]) — the layout kernel without a Buffer."""
    if topk_idx.dtype != torch.int64 or topk_idx.dim() != 2:
        raise ConfigError("topk_idx must be int64 [num_tokens, num_topk]")
    topk_idx = topk_idx.contiguous()
    T, k = topk_idx.shape
    dev = topk_idx.device
    per_rank = torch.empty(num_ranks, dtype=torch.int32, device=dev)
    per_expert = torch.empty(num_experts, dtype=torch.int32, device=dev)
    in_rank = torch.empty((T, num_ranks), dtype=torch.bool, device=dev)
    check(lib.epb_get_dispatch_layout(ptr(topk_idx), T, k, num_experts, num_ranks, ptr(per_rank), ptr(per_expert),
                                      ptr(in_rank), raw_stream()))
    return per_rank, per_expert, in_rank
