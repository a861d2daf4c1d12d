"""Deterministic toy workloads shared by the golden generator and the tests.

Config (BASELINE.json configs[0]): 4 ranks, 128 tokens/rank, hidden 1024,
32 experts, top-2, bf16.  Inputs come from numpy's PCG64 so they regenerate
bit-identically anywhere.  The message plans restate the SPEC's delivery
protocols:

* HT: one WRITE per (token, distinct destination rank) into
  the destination's receive area at ``T*row + src*T*row + pos*row`` (pos =
  rank of the token among the source's tokens for that destination), HT imm
  with a per-(src, dst, channel) sequence; a tail ATOMIC
  (``ht_atomic_operand(False, n)``) after every 32 rows of a channel.
* LL: one WRITE per (token, expert) into
  ``T*row + (le*EP*T + src*T + ordinal)*row``; after a source's last write to
  an expert, a standalone fence ATOMIC with X = that source's count.
Delivery order is scrambled: each message is delayed past later ones with
probability 0.5.
"""
from __future__ import annotations

import hashlib

import numpy as np

EP, T, H, E, K = 4, 128, 1024, 32, 2
ROW = 2 * H
NCH = 4
CHUNK = 32


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def bf16_bits_from_normal(g: np.random.Generator, shape) -> np.ndarray:
    f = g.standard_normal(shape).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    return ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)).astype(np.uint16)


def make_inputs(seed: int = 0, ep=EP, t=T, h=H, e=E, k=K):
    """Per rank: x bf16 bits [t, h], topk_idx int64 [t, k] (distinct experts), weights f32 [t, k]."""
    g = rng(seed)
    xs, idxs, ws = [], [], []
    for _ in range(ep):
        xs.append(bf16_bits_from_normal(g, (t, h)))
        idxs.append(np.argsort(g.random((t, e)), axis=1)[:, :k].astype(np.int64))
        w = g.standard_normal((t, k)).astype(np.float32)
        w = np.exp(w - w.max(axis=1, keepdims=True))
        ws.append((w / w.sum(axis=1, keepdims=True)).astype(np.float32))
    return xs, idxs, ws


def _scramble(g, n):
    t_post = np.arange(n, dtype=np.int64) * 10
    delay = np.where(g.random(n) < 0.5, g.integers(1, 60, n) * 10 + 5, 0)
    t_del = t_post + delay
    order = np.lexsort((np.arange(n), t_del))
    return t_del, order


def _pack_msgs(cols, order, t_del):
    out = {k: np.asarray(v, np.int64)[order] for k, v in cols.items()}
    out["t_del"] = np.asarray(t_del, np.int64)[order]
    return out


def regions_init(xs, recv_rows):
    region_len = T * ROW + recv_rows * ROW
    regions = np.zeros((EP, region_len), np.uint8)
    for s in range(EP):
        regions[s, : T * ROW] = xs[s].view(np.uint8).reshape(-1)
    return regions


def ht_plan(xs, idxs, seed: int = 1):
    """Messages of the HT dispatch delivery (see module doc)."""
    from oracle.codec import encode_ht, ht_atomic_operand
    L = E // EP
    cols = {k: [] for k in ("src", "dst", "src_off", "dst_off", "length", "op_hw", "imm", "work")}
    seq = np.zeros((EP, EP, NCH), np.int64)
    work = 0
    per_ch = T // NCH
    for s in range(EP):
        in_rank = np.zeros((T, EP), bool)
        for j in range(K):
            in_rank[np.arange(T), idxs[s][:, j] // L] = True
        for d in range(EP):
            pos = np.cumsum(in_rank[:, d]) - 1
            for ch in range(NCH):
                toks = [t for t in range(ch * per_ch, (ch + 1) * per_ch) if in_rank[t, d]]
                for c0 in range(0, len(toks), CHUNK):
                    chunk = toks[c0:c0 + CHUNK]
                    for t in chunk:
                        cols["src"].append(s); cols["dst"].append(d)
                        cols["src_off"].append(t * ROW)
                        cols["dst_off"].append(T * ROW + (s * T + int(pos[t])) * ROW)
                        cols["length"].append(ROW); cols["op_hw"].append(0)
                        cols["imm"].append(encode_ht(0, ch, int(seq[s, d, ch]), 0))
                        cols["work"].append(work); work += 1
                        seq[s, d, ch] += 1
                    cols["src"].append(s); cols["dst"].append(d)
                    cols["src_off"].append(0); cols["dst_off"].append(0)
                    cols["length"].append(0); cols["op_hw"].append(0)
                    cols["imm"].append(encode_ht(1, ch, int(seq[s, d, ch]), ht_atomic_operand(False, len(chunk))))
                    cols["work"].append(work); work += 1
                    seq[s, d, ch] += 1
    g = rng(seed)
    n = len(cols["src"])
    t_del, order = _scramble(g, n)
    return _pack_msgs(cols, order, t_del), order


def ll_plan(xs, idxs, seed: int = 2):
    """Messages of the LL dispatch delivery (see module doc)."""
    from oracle.codec import encode_ll
    L = E // EP
    cols = {k: [] for k in ("src", "dst", "src_off", "dst_off", "length", "op_hw", "imm", "work")}
    work = 0
    for s in range(EP):
        for e in range(E):
            d, le = e // L, e % L
            toks = np.nonzero((idxs[s] == e).any(axis=1))[0]
            for ordinal, t in enumerate(toks):
                cols["src"].append(s); cols["dst"].append(d)
                cols["src_off"].append(int(t) * ROW)
                cols["dst_off"].append(T * ROW + (le * EP * T + s * T + ordinal) * ROW)
                cols["length"].append(ROW); cols["op_hw"].append(0)
                cols["imm"].append(encode_ll(0, le, 0))
                cols["work"].append(work); work += 1
            cols["src"].append(s); cols["dst"].append(d)
            cols["src_off"].append(0); cols["dst_off"].append(0)
            cols["length"].append(0); cols["op_hw"].append(0)
            cols["imm"].append(encode_ll(1, le, len(toks)))
            cols["work"].append(work); work += 1
    g = rng(seed)
    n = len(cols["src"])
    t_del, order = _scramble(g, n)
    return _pack_msgs(cols, order, t_del), order


def ht_recv_blocks(regions, idxs):
    """digest[s, d] of the rows source s delivered into d's receive area."""
    L = E // EP
    out = np.zeros((EP, EP, 32), np.uint8)
    for s in range(EP):
        in_rank = np.zeros((T, EP), bool)
        for j in range(K):
            in_rank[np.arange(T), idxs[s][:, j] // L] = True
        for d in range(EP):
            n = int(in_rank[:, d].sum())
            off = T * ROW + s * T * ROW
            out[s, d] = np.frombuffer(hashlib.sha256(regions[d, off: off + n * ROW].tobytes()).digest(), np.uint8)
    return out


def ll_recv_blocks(regions, idxs):
    """digest[d, le] of the rows of local expert le at d, sources ascending, valid slots only."""
    L = E // EP
    out = np.zeros((EP, L, 32), np.uint8)
    for d in range(EP):
        for le in range(L):
            e = d * L + le
            h = hashlib.sha256()
            for s in range(EP):
                n = int((idxs[s] == e).any(axis=1).sum())
                off = T * ROW + (le * EP * T + s * T) * ROW
                h.update(regions[d, off: off + n * ROW].tobytes())
            out[d, le] = np.frombuffer(h.digest(), np.uint8)
    return out


def msgs_digest(msgs) -> np.ndarray:
    h = hashlib.sha256()
    for k in sorted(msgs):
        h.update(k.encode())
        h.update(np.ascontiguousarray(msgs[k], np.int64).tobytes())
    return np.frombuffer(h.digest(), np.uint8)


def digest_rows(rows: np.ndarray) -> np.ndarray:
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(rows).tobytes()).digest(), np.uint8)
