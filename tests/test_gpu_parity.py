"""GPU parity: every device kernel (through the C ABI) against the CPU oracle.

Multi-rank routing is exercised on one GPU with LocalGroup (R ranks in one
process, one kernel launch over all ranks).  Integer/byte outputs must be
bit-exact; combine outputs are also bit-exact here (canonical fp32 order) and
additionally checked against the north-star tolerance rtol 1e-2 / atol 1e-3.
"""
import numpy as np
import pytest

from oracle import ep as O
from tests.golden import toy
from tests.helpers import bf16_bits, bf16_random, make_routing, to_dev_bf16, u8_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    assert _t.cuda.is_available()
    return _t


def _layout_dev(torch, grp_or_buf, idxs, E):
    from paper_2512_19849_b200 import LocalGroup
    dev = [torch.from_numpy(i).cuda() for i in idxs]
    if isinstance(grp_or_buf, LocalGroup):
        return dev, grp_or_buf.get_dispatch_layout(dev, E)
    return dev, [grp_or_buf.get_dispatch_layout(dev[0], E)[:4]]


@pytest.mark.parametrize("R,T,E,k,mask", [(1, 777, 64, 8, 0.0), (4, 1000, 64, 6, 0.1), (8, 4096, 256, 8, 0.0),
                                          (2, 0, 16, 2, 0.0), (8, 5, 32, 32, 0.3)])
def test_layout_parity(torch, R, T, E, k, mask):
    from paper_2512_19849_b200.ops import get_dispatch_layout
    g = np.random.default_rng(R * 1000 + T)
    idx, _ = make_routing(g, T, E, min(k, E), mask)
    per_rank, per_expert, in_rank = get_dispatch_layout(torch.from_numpy(idx).cuda(), E, R)
    torch.cuda.synchronize()
    o_rank, o_exp, o_in = O.get_dispatch_layout(idx, E, R)
    assert np.array_equal(per_rank.cpu().numpy(), o_rank)
    assert np.array_equal(per_expert.cpu().numpy(), o_exp)
    assert np.array_equal(in_rank.cpu().numpy(), o_in)


def _emulated_dispatch(torch, R, Ts, H, E, k, seed, fp8=False, mask=0.0, zipf=0.0, num_sms=None, slots=3,
                       ht="nvlink", grp=None):
    from paper_2512_19849_b200 import Config, LocalGroup
    g = np.random.default_rng(seed)
    xs, idxs, ws = [], [], []
    for r in range(R):
        idx, w = make_routing(g, Ts[r], E, k, mask, zipf)
        xs.append(bf16_random(g, (Ts[r], H)))
        idxs.append(idx)
        ws.append(w)
    from paper_2512_19849_b200 import nvl_bytes_hint, ring_nvl_bytes
    if grp is None and ht == "ring":  # bounded rings of 64 slots: the chunks wrap and wait for credit
        lanes = min(16, 148 // (2 * R))
        grp = LocalGroup(R, ring_nvl_bytes(H, R, k, lanes, 64), ht_transport="ring", ring_lanes=lanes)
    if grp is None:
        grp = LocalGroup(R, nvl_bytes_hint(max(Ts), H, R, k, slots, ht_proxy=ht == "proxy"), num_recv_slots=slots,
                         fifo_channels=4 if ht == "proxy" else 0, proxy_threads=2, ht_transport=ht)
    topk_dev, lay = _layout_dev(torch, grp, idxs, E)
    x_dev = [to_dev_bf16(x) for x in xs]
    scales = None
    if fp8:
        from paper_2512_19849_b200 import per_token_cast_to_fp8
        q = [per_token_cast_to_fp8(x) for x in x_dev]
        x_in = q
        scales = [s.cpu().numpy() for _, s in q]
    else:
        x_in = x_dev
    w_dev = [torch.from_numpy(w).cuda() for w in ws]
    res = grp.dispatch(x_in, [l[3] for l in lay], [l[2] for l in lay], topk_dev, w_dev,
                       config=Config(num_sms) if num_sms else None)
    torch.cuda.synchronize()
    return grp, xs, idxs, ws, x_in, scales, lay, res


@pytest.mark.parametrize("R,Ts,H,E,k,mask,sms,ht", [
    (1, [300], 1024, 16, 4, 0.0, None, "nvlink"),
    (1, [777], 2048, 16, 4, 0.3, None, "nvlink"),  # single-rank path with fully masked tokens
    (2, [257, 64], 2048, 32, 4, 0.0, 7, "nvlink"),
    (4, [128, 128, 128, 128], 1024, 32, 2, 0.0, None, "nvlink"),
    (4, [0, 333, 1, 50], 7168, 64, 8, 0.2, 20, "nvlink"),
    (8, [200] * 8, 1024, 64, 8, 0.0, None, "nvlink"),
    # the CPU-proxy data path (WRITE/ATOMIC TransferCmds)
    (2, [257, 64], 2048, 32, 4, 0.0, 7, "proxy"),
    (4, [0, 333, 1, 50], 7168, 64, 8, 0.2, 20, "proxy"),
    (8, [200] * 8, 1024, 64, 8, 0.0, None, "proxy"),
    # bounded chunked ring channels
    (1, [3000], 1024, 16, 4, 0.0, None, "ring"),
    (2, [2500, 700], 2048, 32, 4, 0.0, 7, "ring"),
    (4, [0, 1333, 1, 900], 7168, 64, 8, 0.2, 20, "ring"),
    (8, [600] * 8, 1024, 64, 8, 0.0, None, "ring"),
])
def test_dispatch_combine_emulated(torch, R, Ts, H, E, k, mask, sms, ht):
    grp = None
    # proxy / ring: the cumulative signal and ring counters must stay in step across calls
    for it in range({"proxy": 2, "ring": 3}.get(ht, 1)):
        grp, xs, idxs, ws, x_in, _, lay, res = _emulated_dispatch(torch, R, Ts, H, E, k, seed=R * 7 + H + it,
                                                                  mask=mask, num_sms=sms, ht=ht, grp=grp)
        _check_dispatch_combine(torch, grp, R, E, xs, idxs, ws, res)
    grp.check_device_error()
    grp.destroy()


def _check_dispatch_combine(torch, grp, R, E, xs, idxs, ws, res):
    in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
    out, heads = O.dispatch(xs, in_ranks, idxs, ws, E)
    for d in range(R):
        recv_x, recv_ti, recv_tw, per_exp, handle = res[d]
        o = out[d]
        assert np.array_equal(bf16_bits(recv_x), o["recv_x"]), d
        assert np.array_equal(recv_ti.cpu().numpy(), o["recv_topk_idx"])
        assert np.array_equal(recv_tw.cpu().numpy(), o["recv_topk_weights"])
        assert np.array_equal(handle[3].cpu().numpy(), o["recv_src_idx"])
        assert np.array_equal(handle[0].cpu().numpy(), o["rank_prefix_matrix"])
        assert per_exp == o["num_recv_per_expert"]
        assert np.array_equal(handle[5].cpu().numpy(), heads[d])
    # combine 1: identity experts (x = recv_x): sum over ranks == x * |ranks|
    comb = grp.combine([r[0] for r in res], [r[4] for r in res], [r[2] for r in res])
    torch.cuda.synchronize()
    ref = O.combine([o["recv_x"] for o in out], in_ranks, heads, out[0]["rank_prefix_matrix"],
                    [o["recv_topk_weights"] for o in out])
    for s in range(R):
        assert np.array_equal(bf16_bits(comb[s][0]), ref[s][0]), s
        assert np.array_equal(comb[s][1].cpu().numpy(), ref[s][1])
        assert np.allclose(comb[s][1].cpu().numpy(), np.where(idxs[s] >= 0, ws[s], 0), atol=0)
    # combine 2: different per-rank expert outputs; bit-exact vs oracle + north-star tolerance
    g = np.random.default_rng(99)
    ys = [bf16_random(g, o["recv_x"].shape) for o in out]
    comb = grp.combine([to_dev_bf16(y) for y in ys], [r[4] for r in res])
    torch.cuda.synchronize()
    ref = O.combine(ys, in_ranks, heads, out[0]["rank_prefix_matrix"])
    for s in range(R):
        got = bf16_bits(comb[s][0])
        assert np.array_equal(got, ref[s][0]), s
        np.testing.assert_allclose(O.bf16_to_f32(got), O.bf16_to_f32(ref[s][0]), rtol=1e-2, atol=1e-3)
        assert comb[s][1] is None


@pytest.mark.parametrize("ht", ["nvlink", "proxy", "ring"])
def test_dispatch_fp8_tuple_emulated(torch, ht):
    R, Ts, H, E, k = 4, [100, 90, 80, 70], 7168, 32, 8
    grp, xs, idxs, ws, x_in, scales, lay, res = _emulated_dispatch(torch, R, Ts, H, E, k, seed=5, fp8=True, ht=ht)
    in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
    qs = [u8_bits(q) for q, _ in x_in]
    out, _ = O.dispatch(qs, in_ranks, idxs, ws, E, x_scales=scales)
    for d in range(R):
        (rx, rs), ti, tw, per_exp, handle = res[d]
        assert rx.dtype == torch.float8_e4m3fn
        assert np.array_equal(u8_bits(rx), out[d]["recv_x"])
        assert np.array_equal(rs.cpu().numpy(), out[d]["recv_scales"])
    grp.destroy()


def test_dispatch_matches_reference_golden_toy(torch):
    """LocalGroup(4) on the toy config reproduces the bytes the reference's
    apply_deliveries put into every (source, destination) block."""
    from pathlib import Path
    from paper_2512_19849_b200 import LocalGroup
    d = np.load(Path(__file__).resolve().parent / "golden" / "ht_dispatch.npz")
    xs, idxs, ws = toy.make_inputs(0)
    grp = LocalGroup(toy.EP, 64 << 20)
    topk_dev, lay = _layout_dev(torch, grp, idxs, toy.E)
    res = grp.dispatch([to_dev_bf16(x) for x in xs], [l[3] for l in lay], [l[2] for l in lay], topk_dev,
                       [torch.from_numpy(w).cuda() for w in ws])
    torch.cuda.synchronize()
    for dst in range(toy.EP):
        rx = bf16_bits(res[dst][0])
        rpm = res[dst][4][0].cpu().numpy()
        for s in range(toy.EP):
            lo = rpm[s - 1, dst] if s else 0
            assert np.array_equal(toy.digest_rows(rx[lo: rpm[s, dst]]), d["blocks"][s, dst])
    grp.destroy()


def test_recv_slot_leases_and_copy_out(torch):
    """recv tensors are zero-copy views of leased slots; when every slot is held the
    scratch slot + copy-out keeps results correct; dropping a view returns its slot."""
    R, Ts, H, E, k = 2, [64, 64], 1024, 8, 2
    grp, xs, idxs, ws, x_in, _, lay, res = _emulated_dispatch(torch, R, Ts, H, E, k, seed=1, slots=2)
    held = [res]
    in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
    out, _ = O.dispatch(xs, in_ranks, idxs, ws, E)
    topk_dev = [torch.from_numpy(i).cuda() for i in idxs]
    for _ in range(3):  # only one leasable slot per rank: these go through the scratch slot
        r2 = grp.dispatch([to_dev_bf16(x) for x in xs], [l[3] for l in lay], [l[2] for l in lay], topk_dev,
                          [torch.from_numpy(w).cuda() for w in ws])
        held.append(r2)
    torch.cuda.synchronize()
    for r in held:
        for d in range(R):
            assert np.array_equal(bf16_bits(r[d][0]), out[d]["recv_x"])
    assert all(rk.num_free_slots() == 0 for rk in grp.ranks)
    del held, res, r2
    import gc
    gc.collect()
    assert all(rk.num_free_slots() == 1 for rk in grp.ranks)
    grp.destroy()


def test_capacity_overflow_raises_config_error(torch):
    from paper_2512_19849_b200 import ConfigError, LocalGroup
    grp = LocalGroup(2, 4 << 20)  # far too small for 4096 x 7168 rows
    g = np.random.default_rng(0)
    idxs = [make_routing(g, 4096, 16, 4)[0] for _ in range(2)]
    topk_dev, lay = _layout_dev(torch, grp, idxs, 16)
    x = [torch.zeros(4096, 7168, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    with pytest.raises(ConfigError):
        grp.dispatch(x, [l[3] for l in lay], [l[2] for l in lay], topk_dev, None)
    # the group stays usable: counters and epochs are in step after the abort
    from paper_2512_19849_b200.errors import EpsimError
    try:
        grp.check_device_error()
    except EpsimError:
        pass
    _, xs, idxs2, ws, _, _, _, res = _emulated_dispatch(torch, 2, [64, 32], 1024, 16, 4, seed=3, grp=grp)
    _check_dispatch_combine(torch, grp, 2, 16, xs, idxs2, ws, res)
    grp.destroy()


@pytest.mark.parametrize("ht", ["nvlink", "ring"])
def test_buffer_single_rank_deepseek_shape(torch, ht):
    """Buffer at N=1 (EP=1) on the DeepSeek-V3 shape: recv_x == x, combine(dispatch(x)) == x
    (the single-rank dispatch path, and the chunked-ring transport)."""
    from paper_2512_19849_b200 import Buffer, nvl_bytes_hint, ring_nvl_bytes
    T, H, E, k = 4096, 7168, 256, 8
    g = np.random.default_rng(42)
    idx, w = make_routing(g, T, E, k)
    x = to_dev_bf16(bf16_random(g, (T, H)))
    nvl = ring_nvl_bytes(H, 1, k) if ht == "ring" else nvl_bytes_hint(T, H, 1, k)
    buf = Buffer(None, nvl, ht_transport=ht)
    topk = torch.from_numpy(idx).cuda()
    wt = torch.from_numpy(w).cuda()
    per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(topk, E)
    recv_x, rti, rtw, lst, handle, _ = buf.dispatch(x, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank,
                                                    num_tokens_per_expert=per_exp, topk_idx=topk, topk_weights=wt)
    assert torch.equal(recv_x, x)
    assert torch.equal(rti, topk) and torch.equal(rtw, wt)
    assert lst == np.bincount(idx.ravel(), minlength=E).tolist()
    out, out_w, _ = buf.combine(recv_x, handle, topk_weights=rtw)
    assert torch.equal(out, x) and torch.equal(out_w, wt)
    # cached-handle dispatch
    rx2, *_ = buf.dispatch(x, handle=handle)
    assert torch.equal(rx2, x)
    buf.destroy()


# --- FP8 cast --------------------------------------------------------------------------
@pytest.mark.parametrize("round_scale", [False, True])
def test_fp8_cast_parity(torch, round_scale):
    from paper_2512_19849_b200 import per_token_cast_to_fp8
    g = np.random.default_rng(8)
    x = bf16_random(g, (333, 7168), scale=3.0)
    x[0, :128] = 0  # amax floor
    x[1, :] = bf16_random(g, (7168,), scale=1e4)  # large values
    q, s = per_token_cast_to_fp8(to_dev_bf16(x), round_scale=round_scale)
    oq, os_ = O.fp8_quant(x, round_scale)
    assert np.array_equal(u8_bits(q), oq)
    assert np.array_equal(s.cpu().numpy(), os_)


# --- low latency -------------------------------------------------------------------------
def _ll_case(torch, R, T, H, E, k, use_fp8, seed, transport="nvlink", round_scale=False, mask=0.0, Tmax=None):
    from paper_2512_19849_b200 import Buffer, LocalGroup
    Tmax = Tmax or max(T, 1)
    g = np.random.default_rng(seed)
    xs, idxs, ws = [], [], []
    for _ in range(R):
        idx, w = make_routing(g, T, E, k, mask)
        idxs.append(idx)
        ws.append(w)
        xs.append(bf16_random(g, (T, H)))
    ll_bytes = Buffer.get_low_latency_rdma_size_hint(Tmax, H, R, E, num_topk=k)
    grp = LocalGroup(R, 1 << 20, ll_bytes, fifo_channels=min(64, 4 * R) if transport == "proxy" else 0, proxy_threads=2,
                     ll_transport=transport)
    res, hook = grp.low_latency_dispatch([to_dev_bf16(x) for x in xs], [torch.from_numpy(i).cuda() for i in idxs],
                                         Tmax, E, use_fp8=use_fp8, round_scale=round_scale)
    torch.cuda.synchronize()
    grp.check_device_error()
    return grp, xs, idxs, ws, res, Tmax


def _check_ll_dispatch(torch, R, E, xs, idxs, res, Tmax, use_fp8, round_scale=False):
    L = E // R
    out, comb_slots = O.ll_dispatch(xs, idxs, E, Tmax, use_fp8=use_fp8, round_scale=round_scale)
    for d in range(R):
        recv, count, handle = res[d]
        src_info, layout_range = handle[0].cpu().numpy(), handle[1].cpu().numpy()
        cnt = count.cpu().numpy()
        if use_fp8:
            rx, rs = recv
            rxb = u8_bits(rx)
            rsn = rs.cpu().numpy()
        else:
            rxb = bf16_bits(recv)
        for le in range(L):
            o = out[d][le]
            n = o["count"]
            assert cnt[le] == n
            assert np.array_equal(src_info[le, :n], o["tok"])
            assert [(int(v) >> 32, int(v) & 0xFFFFFFFF) for v in layout_range[le]] == o["layout"]
            if n:
                assert np.array_equal(rxb[le, :n], o["x"]), (d, le)
                if use_fp8:
                    assert np.array_equal(rsn[le, :n], o["scales"])
    return out, comb_slots


@pytest.mark.parametrize("R,T,H,E,k,fp8,transport", [
    (1, 128, 7168, 32, 8, True, "nvlink"),
    (2, 100, 1024, 16, 4, False, "nvlink"),
    (4, 128, 7168, 32, 8, True, "nvlink"),
    (8, 64, 2048, 64, 8, True, "nvlink"),
    (2, 50, 1024, 16, 4, True, "proxy"),
    (4, 128, 7168, 64, 8, True, "proxy"),
])
def test_ll_dispatch_combine_parity(torch, R, T, H, E, k, fp8, transport):
    grp, xs, idxs, ws, res, Tmax = _ll_case(torch, R, T, H, E, k, fp8, seed=R + T, transport=transport, mask=0.05)
    out, comb_slots = _check_ll_dispatch(torch, R, E, xs, idxs, res, Tmax, fp8)
    L = E // R
    if transport == "nvlink":  # (the proxy transport lays rows out token-major: its slots differ by design)
        for d in range(R):
            assert np.array_equal(res[d][2][6].cpu().numpy(), comb_slots[d])
    # combine: random expert outputs
    g = np.random.default_rng(123)
    ys = [bf16_random(g, (L, R * Tmax, H)) for _ in range(R)]
    comb, _ = grp.low_latency_combine([to_dev_bf16(y) for y in ys], [torch.from_numpy(i).cuda() for i in idxs],
                                      [torch.from_numpy(w).cuda() for w in ws], [r[2] for r in res])
    torch.cuda.synchronize()
    grp.check_device_error()
    expert_outs = [[ys[d][le, : out[d][le]["count"]] for le in range(L)] for d in range(R)]
    ref = O.ll_combine(expert_outs, idxs, ws, E)
    for s in range(R):
        got = bf16_bits(comb[s])
        assert np.array_equal(got, ref[s]), s
        np.testing.assert_allclose(O.bf16_to_f32(got), O.bf16_to_f32(ref[s]), rtol=1e-2, atol=1e-3)
    # a second round on the other parity, with the recv hook split
    res2, hook = grp.low_latency_dispatch([to_dev_bf16(x) for x in xs], [torch.from_numpy(i).cuda() for i in idxs],
                                          Tmax, E, use_fp8=fp8, return_recv_hook=True)
    hook()
    torch.cuda.synchronize()
    _check_ll_dispatch(torch, R, E, xs, idxs, res2, Tmax, fp8)
    grp.destroy()


def test_ll_matches_reference_golden_toy(torch):
    from pathlib import Path
    d = np.load(Path(__file__).resolve().parent / "golden" / "ll_dispatch.npz")
    from paper_2512_19849_b200 import Buffer, LocalGroup
    xs, idxs, _ = toy.make_inputs(0)
    ll_bytes = Buffer.get_low_latency_rdma_size_hint(toy.T, toy.H, toy.EP, toy.E, num_topk=toy.K)
    grp = LocalGroup(toy.EP, 1 << 20, ll_bytes)
    res, _ = grp.low_latency_dispatch([to_dev_bf16(x) for x in xs], [torch.from_numpy(i).cuda() for i in idxs],
                                      toy.T, toy.E, use_fp8=False)
    torch.cuda.synchronize()
    L = toy.E // toy.EP
    for dst in range(toy.EP):
        rx = bf16_bits(res[dst][0])
        cnt = res[dst][1].cpu().numpy()
        for le in range(L):
            assert cnt[le] == d["counters"][dst, le]
            assert np.array_equal(toy.digest_rows(rx[le, : cnt[le]]), d["blocks"][dst, le])
    grp.destroy()


def test_ll_round_scale(torch):
    grp, xs, idxs, ws, res, Tmax = _ll_case(torch, 2, 32, 2048, 16, 4, True, seed=3, round_scale=True)
    _check_ll_dispatch(torch, 2, 16, xs, idxs, res, Tmax, True, round_scale=True)
    grp.destroy()


def test_fifo_device_producer(torch):
    """GPU producer -> pinned FIFO -> CPU proxy (count-only) -> check_completion on the GPU."""
    import ctypes as C
    from paper_2512_19849_b200 import Buffer
    from paper_2512_19849_b200._lib import lib
    buf = Buffer(None, 1 << 20, 1 << 20, low_latency_mode=True, fifo_channels=8, fifo_capacity=256,
                 proxy_threads=4, ll_transport="proxy")
    el = C.c_int64()
    n = 1 << 18
    assert lib.epb_fifo_device_bench(buf._rank.ctx, n, 8, C.byref(el), torch.cuda.current_stream().cuda_stream) == 0
    stats = (C.c_int64 * 3)()
    lib.epb_proxy_stats(buf._rank.ctx, stats)
    assert stats[0] == n
    print(f"device FIFO: {n} cmds over 8 channels in {el.value / 1e3:.1f} us = {n / el.value * 1e3:.1f} Mcmd/s")
    buf.destroy()
