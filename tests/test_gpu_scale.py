"""GPU parity at the benchmarked shapes (BASELINE.json configs 2-5) and soak runs.

Every test runs R = 8 ranks emulated on one GPU (LocalGroup: one symmetric
region per rank, one launch over all ranks) at the exact sizes bench.py times:

* DeepSeek-V3 normal mode, T=4096/rank, H=7168, 256 experts, top-8 — bf16
  dispatch, bf16 combine, and the FP8 (+ per-128-channel scales) dispatch;
* Qwen3-235B-A22B, T=8192/rank, H=4096, 128 experts, top-8, Zipf(1.0) routing;
* DeepSeek-V3 low-latency decode, T=128/rank, H=7168, 256 experts, top-8, FP8,
  over the direct NVLink transport and through the GPU->CPU FIFO + CPU proxy.

Rows are compared block by block against the oracle's receive order
(oracle.ep.recv_order) instead of materialising every destination's rows;
metadata, handles and combine outputs are compared with the full oracle.
The soak tests follow SPEC.md's acceptance criterion 1 (EP=8, top-4, 4096
tokens, many iterations over 20 seeds, bit-exact every iteration) and its
ring-safety invariant (canary per slot, no unread slot
overwritten over 10^4 randomized iterations; SPEC.md:444 zero canary trips).
"""
import os

import numpy as np
import pytest

from oracle import ep as O
from tests.helpers import bf16_bits, make_routing, to_dev_bf16, u8_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    assert _t.cuda.is_available()
    return _t


def _gpu_bf16(torch, gen, shape):
    """Seeded N(0,1) bf16 on the device (fast at GB scale) and its bits on the host."""
    x = torch.randn(shape, generator=gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    return x, bf16_bits(x)


def _routing(R, T, E, k, seed, zipf=0.0):
    idxs, ws = [], []
    for r in range(R):
        g = np.random.default_rng(seed * 1000 + r)
        idx, w = make_routing(g, T, E, k, zipf=zipf)
        idxs.append(idx)
        ws.append(w)
    return idxs, ws


def _check_rows(got_rows, src_rows, in_ranks, d, rpm, what):
    """got_rows: destination d's received rows (host array); src_rows[s]: source s's rows."""
    srcs, toks = O.recv_order(in_ranks, d)
    assert got_rows.shape[0] == len(toks), (what, d, got_rows.shape[0], len(toks))
    R = len(in_ranks)
    for s in range(R):
        lo = int(rpm[s - 1, d]) if s else 0
        hi = int(rpm[s, d])
        assert np.array_equal(got_rows[lo:hi], src_rows[s][toks[lo:hi]]), (what, "dst", d, "src", s)


def _check_meta(res, meta, heads, d, fp8=False):
    recv_x, ti, tw, per_exp, handle = res[d]
    o = meta[d]
    assert np.array_equal(ti.cpu().numpy(), o["recv_topk_idx"]), d
    assert np.array_equal(tw.cpu().numpy(), o["recv_topk_weights"]), d
    assert np.array_equal(handle[3].cpu().numpy(), o["recv_src_idx"]), d
    assert np.array_equal(handle[0].cpu().numpy(), o["rank_prefix_matrix"]), d
    assert per_exp == o["num_recv_per_expert"], d
    assert np.array_equal(handle[5].cpu().numpy(), heads[d]), d


def _normal_full_size(torch, R, T, H, E, k, seed, zipf=0.0, fp8_too=False):
    from paper_2512_19849_b200 import LocalGroup, nvl_bytes_hint, per_token_cast_to_fp8
    idxs, ws = _routing(R, T, E, k, seed, zipf)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    xd, xb = zip(*[_gpu_bf16(torch, gen, (T, H)) for _ in range(R)])
    grp = LocalGroup(R, nvl_bytes_hint(T, H, R, k, num_slots=2), num_recv_slots=2)
    try:
        topk = [torch.from_numpy(i).cuda() for i in idxs]
        wd = [torch.from_numpy(w).cuda() for w in ws]
        lay = grp.get_dispatch_layout(topk, E)
        in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
        for r in range(R):  # the layout kernel at this shape
            o_rank, o_exp, o_in = O.get_dispatch_layout(idxs[r], E, R)
            assert np.array_equal(lay[r][0].cpu().numpy(), o_rank)
            assert np.array_equal(lay[r][2].cpu().numpy(), o_exp)
            assert np.array_equal(lay[r][3].cpu().numpy(), o_in)
        res = grp.dispatch(list(xd), [l[3] for l in lay], [l[2] for l in lay], topk, wd)
        torch.cuda.synchronize()
        grp.check_device_error()
        meta, heads = O.dispatch(None, in_ranks, idxs, ws, E)
        rpm = meta[0]["rank_prefix_matrix"]
        for d in range(R):
            _check_rows(bf16_bits(res[d][0]), xb, in_ranks, d, rpm, "bf16")
            _check_meta(res, meta, heads, d)
        # combine: per-rank random expert outputs; bit-exact vs the canonical-order oracle
        ys = [_gpu_bf16(torch, gen, (res[d][0].shape[0], H)) for d in range(R)]
        comb = grp.combine([y for y, _ in ys], [r[4] for r in res], [r[2] for r in res])
        torch.cuda.synchronize()
        grp.check_device_error()
        ref = O.combine([yb for _, yb in ys], in_ranks, heads, rpm, [m["recv_topk_weights"] for m in meta])
        for s in range(R):
            got = bf16_bits(comb[s][0])
            assert np.array_equal(got, ref[s][0]), ("combine", s)
            np.testing.assert_allclose(O.bf16_to_f32(got), O.bf16_to_f32(ref[s][0]), rtol=1e-2, atol=1e-3)
            assert np.array_equal(comb[s][1].cpu().numpy(), ref[s][1]), ("combine weights", s)
        del ys, comb, res
        if fp8_too:  # config 3: FP8 dispatch with per-128-channel scales on the same routing
            q = [per_token_cast_to_fp8(x) for x in xd]
            oq, osc = O.fp8_quant(xb[0])  # the cast itself, pinned on rank 0's tokens
            assert np.array_equal(u8_bits(q[0][0]), oq)
            assert np.array_equal(q[0][1].cpu().numpy(), osc)
            qb = [u8_bits(a) for a, _ in q]
            sb = [b.cpu().numpy() for _, b in q]
            res = grp.dispatch(q, [l[3] for l in lay], [l[2] for l in lay], topk, wd)
            torch.cuda.synchronize()
            grp.check_device_error()
            for d in range(R):
                (rx, rs), *_ = res[d]
                assert rx.dtype == torch.float8_e4m3fn
                _check_rows(u8_bits(rx), qb, in_ranks, d, rpm, "fp8")
                _check_rows(rs.cpu().numpy(), sb, in_ranks, d, rpm, "scales")
                _check_meta(res, meta, heads, d)
    finally:
        grp.destroy()


def test_dsv3_normal_ep8_full_size(torch):
    """BASELINE configs 2 + 3 at EP=8: T=4096/rank, H=7168, 256 experts, top-8, bf16 and FP8."""
    _normal_full_size(torch, 8, 4096, 7168, 256, 8, seed=11, fp8_too=True)


def test_qwen3_zipf_ep8_full_size(torch):
    """BASELINE config 5 at EP=8: T=8192/rank, H=4096, 128 experts, top-8, Zipf(1.0) popularity."""
    _normal_full_size(torch, 8, 8192, 4096, 128, 8, seed=12, zipf=1.0)


@pytest.mark.parametrize("transport", ["nvlink", "proxy"])
def test_dsv3_ll_ep8_full_size(torch, transport):
    """BASELINE config 4 at EP=8: 128 tokens/rank, H=7168, 256 experts, top-8, FP8 dispatch, bf16 combine."""
    from tests.test_gpu_parity import _check_ll_dispatch, _ll_case
    R, T, H, E, k = 8, 128, 7168, 256, 8
    grp, xs, idxs, ws, res, Tmax = _ll_case(torch, R, T, H, E, k, True, seed=13, transport=transport)
    try:
        out, comb_slots = _check_ll_dispatch(torch, R, E, xs, idxs, res, Tmax, True)
        if transport == "nvlink":  # proxy rows are token-major: different (internal) combine slots
            for d in range(R):
                assert np.array_equal(res[d][2][6].cpu().numpy(), comb_slots[d])
        L = E // R
        gen = torch.Generator(device="cuda")
        gen.manual_seed(13)
        ys = [_gpu_bf16(torch, gen, (L, R * Tmax, H)) for _ in range(R)]
        for it in range(3):  # repeated pairs: device epochs, parities and proxy signal targets stay in step
            comb, _ = grp.low_latency_combine([y for y, _ in ys], [torch.from_numpy(i).cuda() for i in idxs],
                                              [torch.from_numpy(w).cuda() for w in ws], [r[2] for r in res])
            torch.cuda.synchronize()
            grp.check_device_error()
            expert_outs = [[ys[d][1][le, : out[d][le]["count"]] for le in range(L)] for d in range(R)]
            ref = O.ll_combine(expert_outs, idxs, ws, E)
            for s in range(R):
                got = bf16_bits(comb[s])
                assert np.array_equal(got, ref[s]), (it, s)
                np.testing.assert_allclose(O.bf16_to_f32(got), O.bf16_to_f32(ref[s]), rtol=1e-2, atol=1e-3)
            if it < 2:
                res, _ = grp.low_latency_dispatch([to_dev_bf16(x) for x in xs],
                                                  [torch.from_numpy(i).cuda() for i in idxs], Tmax, E, use_fp8=True)
                torch.cuda.synchronize()
                _check_ll_dispatch(torch, R, E, xs, idxs, res, Tmax, True)
    finally:
        grp.destroy()


def test_soak_ep8_top4_bitexact(torch):
    """SPEC.md acceptance criterion 1 on the device path: EP=8, top-4, 4096 tokens/rank,
    20 seeds x EPB_SOAK_ITERS/20 iterations (default 200 calls; EPB_SOAK_ITERS=1000 is the full criterion), fresh routing
    every call on one long-lived group, dispatch and combine bit-exact every call."""
    from paper_2512_19849_b200 import LocalGroup, nvl_bytes_hint
    R, T, H, E, k = 8, 4096, 256, 64, 4
    total = int(os.environ.get("EPB_SOAK_ITERS", "200"))
    seeds = 20
    per_seed = max(1, total // seeds)
    grp = LocalGroup(R, nvl_bytes_hint(T, H, R, k, num_slots=2), num_recv_slots=2)
    calls = 0
    try:
        for seed in range(seeds):
            g = np.random.default_rng(1000 + seed)
            gen = torch.Generator(device="cuda")
            gen.manual_seed(1000 + seed)
            for it in range(per_seed):
                idxs, ws = [], []
                for r in range(R):
                    idx, w = make_routing(g, T, E, k, mask_frac=0.02 if it % 3 == 0 else 0.0)
                    idxs.append(idx)
                    ws.append(w)
                xd, xb = zip(*[_gpu_bf16(torch, gen, (T, H)) for _ in range(R)])
                topk = [torch.from_numpy(i).cuda() for i in idxs]
                lay = grp.get_dispatch_layout(topk, E)
                res = grp.dispatch(list(xd), [l[3] for l in lay], [l[2] for l in lay], topk,
                                   [torch.from_numpy(w).cuda() for w in ws])
                # per-expert affine stamp (SPEC.md design decision: out = in + expert stamp):
                # a mis-routed row combines to a different value
                ys = [(r[0].float() + float(d + 1)).to(torch.bfloat16) for d, r in enumerate(res)]
                comb = grp.combine(ys, [r[4] for r in res], [r[2] for r in res])
                torch.cuda.synchronize()
                in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
                meta, heads = O.dispatch(None, in_ranks, idxs, ws, E)
                rpm = meta[0]["rank_prefix_matrix"]
                ys_b = []
                for d in range(R):
                    _check_rows(bf16_bits(res[d][0]), xb, in_ranks, d, rpm, f"seed {seed} it {it}")
                    _check_meta(res, meta, heads, d)
                    ys_b.append(bf16_bits(ys[d]))
                ref = O.combine(ys_b, in_ranks, heads, rpm, [m["recv_topk_weights"] for m in meta])
                for s in range(R):
                    assert np.array_equal(bf16_bits(comb[s][0]), ref[s][0]), ("combine", seed, it, s)
                    assert np.array_equal(comb[s][1].cpu().numpy(), ref[s][1]), ("weights", seed, it, s)
                calls += 1
        grp.check_device_error()
    finally:
        grp.destroy()
    assert calls == seeds * per_seed


def _ring_group(R, H, k, lanes, ring_tokens=64):
    from paper_2512_19849_b200 import LocalGroup, ring_nvl_bytes
    return LocalGroup(R, ring_nvl_bytes(H, R, k, lanes, ring_tokens), ht_transport="ring", ring_lanes=lanes)


def test_ring_canary_soak(torch):
    """Ring safety: every ring slot carries a canary (its cumulative
    sequence number); the receiver checks it before and after reading the slot.
    EPB_RING_ITERS (default 10^4) randomized ring dispatch+combine calls on 64-slot
    rings that wrap many times per call: zero canary trips, and the outputs stay
    bit-exact (checked against the oracle every 200th call and on the last)."""
    from paper_2512_19849_b200 import LocalGroup  # noqa: F401
    R, H, E, k, lanes = 4, 128, 32, 4, 4
    iters = int(os.environ.get("EPB_RING_ITERS", "10000"))
    grp = _ring_group(R, H, k, lanes)
    g = np.random.default_rng(77)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(77)
    try:
        for it in range(iters):
            Ts = [int(t) for t in g.integers(0, 700, R)]
            idxs, ws = [], []
            for r in range(R):
                idx, w = make_routing(g, Ts[r], E, k, mask_frac=0.05)
                idxs.append(idx)
                ws.append(w)
            xd = [torch.randn((Ts[r], H), generator=gen, device="cuda").to(torch.bfloat16) for r in range(R)]
            topk = [torch.from_numpy(i).cuda() for i in idxs]
            lay = grp.get_dispatch_layout(topk, E)
            res = grp.dispatch(xd, [l[3] for l in lay], [l[2] for l in lay], topk,
                               [torch.from_numpy(w).cuda() for w in ws])
            comb = grp.combine([r[0] for r in res], [r[4] for r in res], [r[2] for r in res])
            grp.check_device_error()  # raises InvariantViolation on a canary trip
            if it % 200 == 0 or it == iters - 1:
                torch.cuda.synchronize()
                xb = [bf16_bits(x) for x in xd]
                in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
                out, heads = O.dispatch(xb, in_ranks, idxs, ws, E)
                for d in range(R):
                    assert np.array_equal(bf16_bits(res[d][0]), out[d]["recv_x"]), (it, d)
                    assert np.array_equal(res[d][4][3].cpu().numpy(), out[d]["recv_src_idx"]), (it, d)
                ref = O.combine([o["recv_x"] for o in out], in_ranks, heads, out[0]["rank_prefix_matrix"],
                                [o["recv_topk_weights"] for o in out])
                for s in range(R):
                    assert np.array_equal(bf16_bits(comb[s][0]), ref[s][0]), (it, s)
        torch.cuda.synchronize()
        grp.check_device_error()
    finally:
        grp.destroy()


def test_ring_canary_catches_overrun(torch, monkeypatch):
    """The canaries are live: with the sender's credit wait disabled
    (EPB_RING_UNSAFE_NO_CREDIT=1, a test hook) the sender overruns unread slots of
    a 64-slot ring and the receiver reports InvariantViolation instead of
    delivering overwritten rows."""
    from paper_2512_19849_b200.errors import EpsimError, InvariantViolation
    R, T, H, E, k, lanes = 2, 4000, 1024, 16, 4, 1
    grp = _ring_group(R, H, k, lanes)
    monkeypatch.setenv("EPB_RING_UNSAFE_NO_CREDIT", "1")
    try:
        g = np.random.default_rng(5)
        idxs = [make_routing(g, T, E, k)[0] for _ in range(R)]
        xd = [torch.randn((T, H), device="cuda").to(torch.bfloat16) for _ in range(R)]
        topk = [torch.from_numpy(i).cuda() for i in idxs]
        lay = grp.get_dispatch_layout(topk, E)
        grp.dispatch(xd, [l[3] for l in lay], [l[2] for l in lay], topk, None)
        torch.cuda.synchronize()
        with pytest.raises(InvariantViolation):
            grp.check_device_error()
    finally:
        monkeypatch.delenv("EPB_RING_UNSAFE_NO_CREDIT")
        try:
            grp.check_device_error()
        except EpsimError:
            pass
        grp.destroy()
