"""Shared helpers for the GPU parity tests (numpy <-> torch, seeded inputs)."""
from __future__ import annotations

import numpy as np


def to_dev_bf16(u16: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(u16).view(np.int16)).view(torch.bfloat16).cuda()


def bf16_bits(t) -> np.ndarray:
    import torch
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def u8_bits(t) -> np.ndarray:
    import torch
    return t.detach().contiguous().view(torch.uint8).cpu().numpy()


def make_routing(g: np.random.Generator, T: int, E: int, k: int, mask_frac: float = 0.0, zipf: float = 0.0):
    """Distinct experts per token; optional masked (-1) entries and Zipf-skewed popularity."""
    if zipf > 0:
        p = 1.0 / np.arange(1, E + 1) ** zipf
        perm = g.permutation(E)
        pop = np.empty(E)
        pop[perm] = p / p.sum()
        # k draws without replacement with probability ~ pop: the top-k of
        # log(pop) + Gumbel noise (the Gumbel-top-k trick), vectorised over tokens
        key = np.log(pop)[None, :] - np.log(-np.log(g.random((T, E))))
        idx = np.argsort(-key, axis=1)[:, :k] if T else np.zeros((0, k), int)
    else:
        idx = np.argsort(g.random((T, E)), axis=1)[:, :k] if T else np.zeros((0, k), int)
    idx = idx.astype(np.int64)
    if mask_frac > 0 and T:
        idx[g.random((T, k)) < mask_frac] = -1
    w = g.random((T, k)).astype(np.float32) + np.float32(0.05)
    w = (w / w.sum(axis=1, keepdims=True)).astype(np.float32)
    return idx, w


def bf16_random(g: np.random.Generator, shape, scale=1.0) -> np.ndarray:
    f = (g.standard_normal(shape) * scale).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    return ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)).astype(np.uint16)
