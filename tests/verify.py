"""Oracle verification of one benchmarked step — TEST INFRASTRUCTURE.

bench.py calls these OUTSIDE its timed regions (one step per configuration)
to mark each bench entry ``"verified": true``.  Every rank checks what it
received and what it combined, regenerating the other ranks' seeded inputs
(device RNG for the rows, numpy for the routing) so no data is exchanged.

* normal mode: received rows (per source block, in the oracle's receive
  order), FP8 bytes and scales, top-k indices / weights, source indices, the
  rank prefix matrix, per-expert counts, send_head; combine of this rank's
  tokens against oracle.ep.combine_rank (canonical fp32 order, one bf16 RNE);
* low latency: per-expert counts, packed rows (FP8 bytes + scales), src_info,
  layout ranges, and the LL combine against oracle.ep.ll_combine.
"""
from __future__ import annotations

import numpy as np

from oracle import ep as O
from tests.helpers import bf16_bits, make_routing, u8_bits


def seeded_x(torch, seed: int, T: int, H: int, dev):
    """N(0,1) bf16 rows from a seeded device generator (any rank can regenerate them)."""
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    return torch.randn((T, H), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)


def routing(seed: int, T: int, E: int, k: int, zipf: float = 0.0):
    return make_routing(np.random.default_rng(int(seed)), T, E, k, zipf=zipf)


def _rows_equal(torch, got, src, toks_np):
    t_idx = torch.from_numpy(np.ascontiguousarray(toks_np, np.int64)).to(got.device)
    exp = src.index_select(0, t_idx)
    return torch.equal(got.contiguous().view(torch.uint8), exp.contiguous().view(torch.uint8))


def verify_normal(torch, rank, R, E, inputs, res, comb, *, fp8_cast=None, check_tokens=None, check_per_expert=True):
    """inputs(s) -> (x bf16, idx, w): source s's tokens and routing; fp8_cast:
    the FP8 cast the dispatch input went through (None for bf16 dispatch).  res: this rank's Buffer.dispatch result
    (recv_x, topk_idx, topk_w, per-expert list, handle); comb: (combined_x,
    combined_w) of combining the received rows back (identity experts; FP8
    rows are cast to bf16 first).  Raises AssertionError on any mismatch."""
    fp8 = fp8_cast is not None
    srcs = []
    for s in range(R):
        x, i, w = inputs(s)
        srcs.append(((fp8_cast(x) if fp8 else x), i, w, x))
    idxs = [s[1] for s in srcs]
    ws = [s[2] for s in srcs]
    in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
    meta, heads = O.dispatch(None, in_ranks, idxs, ws, E)
    rpm = meta[0]["rank_prefix_matrix"]
    o = meta[rank]
    recv_x, ti, tw, per_exp, handle = res
    rx = recv_x[0] if fp8 else recv_x
    _, toks = O.recv_order(in_ranks, rank)
    assert rx.shape[0] == len(toks), ("rows", rx.shape[0], len(toks))
    for s in range(R):
        lo, hi = (int(rpm[s - 1, rank]) if s else 0), int(rpm[s, rank])
        src = srcs[s][0][0] if fp8 else srcs[s][0]
        assert _rows_equal(torch, rx[lo:hi], src, toks[lo:hi]), ("rows from source", s)
        if fp8:
            assert _rows_equal(torch, recv_x[1][lo:hi], srcs[s][0][1], toks[lo:hi]), ("scales from source", s)
    if ti is not None:
        assert np.array_equal(ti.cpu().numpy(), o["recv_topk_idx"]), "recv_topk_idx"
        assert np.array_equal(tw.cpu().numpy(), o["recv_topk_weights"]), "recv_topk_weights"
        if check_per_expert:
            assert per_exp == o["num_recv_per_expert"], "num_recv_tokens_per_expert"
    assert np.array_equal(handle[3].cpu().numpy(), o["recv_src_idx"]), "recv_src_idx"
    assert np.array_equal(handle[0].cpu().numpy(), rpm), "rank_prefix_matrix"
    assert np.array_equal(handle[5].cpu().numpy(), heads[rank]), "send_head"
    if fp8:  # the cast itself, on a slice of this rank's tokens
        x_bf16 = srcs[rank][3]
        n8 = min(64, x_bf16.shape[0])
        oq, osc = O.fp8_quant(bf16_bits(x_bf16[:n8]))
        assert np.array_equal(u8_bits(srcs[rank][0][0][:n8]), oq), "fp8 cast"
        assert np.array_equal(srcs[rank][0][1][:n8].cpu().numpy(), osc), "fp8 scales"
    # combine of this rank's (first check_tokens) tokens: every destination's
    # expert output for them is the row it received (cast to bf16 for FP8)
    T = in_ranks[rank].shape[0]
    n = T if check_tokens is None else min(T, int(check_tokens))
    mine = srcs[rank][0][0] if fp8 else srcs[rank][0]
    if fp8:
        y_mine = O.f32_to_bf16(O.e4m3_decode(u8_bits(mine[:n])))
    else:
        y_mine = bf16_bits(mine[:n])
    H = y_mine.shape[1] if n else rx.shape[1]
    recv_xs, recv_ws = [], []
    ir, sh = in_ranks[rank][:n], heads[rank][:n]
    for d in range(R):
        nd = int(rpm[R - 1, d])
        ys = np.zeros((nd, H), np.uint16)
        t_sel = np.nonzero(ir[:, d])[0]
        base = int(rpm[rank - 1, d]) if rank else 0
        ys[base + sh[t_sel, d]] = y_mine[t_sel]
        recv_xs.append(ys)
        recv_ws.append(meta[d]["recv_topk_weights"])
    exp_x, exp_w = O.combine_rank(rank, recv_xs, ir, sh, rpm, recv_ws if comb[1] is not None else None)
    assert np.array_equal(bf16_bits(comb[0][:n]), exp_x), "combined_x"
    if comb[1] is not None:
        assert np.array_equal(comb[1][:n].cpu().numpy(), exp_w), "combined_topk_weights"
    return {"tokens_combined_checked": n, "rows_checked": int(len(toks))}


def verify_ll(torch, rank, R, E, Tmax, inputs, ys, recv, count, handle, combined):
    """inputs(s) -> (x bf16 tensor, idx, w); ys(d) -> expert outputs [L, R*Tmax, H] of rank d.
    recv = (fp8 rows, scales); count, handle: this rank's low_latency_dispatch outputs;
    combined: this rank's low_latency_combine output."""
    srcs = [inputs(s) for s in range(R)]
    xs = [bf16_bits(s[0]) for s in srcs]
    idxs = [s[1] for s in srcs]
    ws = [s[2] for s in srcs]
    out, comb_slots = O.ll_dispatch(xs, idxs, E, Tmax, use_fp8=True)
    L = E // R
    q, sc = u8_bits(recv[0]), recv[1].cpu().numpy()
    cnt = count.cpu().numpy()
    src_info, layout_range = handle[0].cpu().numpy(), handle[1].cpu().numpy()
    for le in range(L):
        ob = out[rank][le]
        n = ob["count"]
        assert cnt[le] == n, ("count", le)
        assert np.array_equal(src_info[le, :n], ob["tok"]), ("src_info", le)
        assert [(int(v) >> 32, int(v) & 0xFFFFFFFF) for v in layout_range[le]] == ob["layout"], ("layout", le)
        if n:
            assert np.array_equal(q[le, :n], ob["x"]), ("fp8 rows", le)
            assert np.array_equal(sc[le, :n], ob["scales"]), ("scales", le)
    if not handle[9]:  # direct transport: expert-major rows, the oracle's slots (proxy rows are token-major)
        assert np.array_equal(handle[6].cpu().numpy(), comb_slots[rank]), "combine slots"
    expert_outs = []
    for d in range(R):
        y = ys(d)
        expert_outs.append([bf16_bits(y[le, : out[d][le]["count"]]) for le in range(L)])
    ref = O.ll_combine(expert_outs, idxs, ws, E)
    assert np.array_equal(bf16_bits(combined), ref[rank]), "ll combined"
    return {"messages_checked": int(sum(out[rank][le]["count"] for le in range(L)))}
