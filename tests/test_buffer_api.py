"""DeepEP drop-in surface of Buffer beyond the basic calls ("without
any line of code change"): num_worst_tokens (no host sync) and CUDA-graph
capture of layout -> dispatch -> combine, the comm stream behind
previous_event / async_finish / allocate_on_comm_stream, and the zero-copy
low-latency combine buffer.  Every output is checked against the oracle."""
import numpy as np
import pytest

from oracle import ep as O
from tests.helpers import bf16_bits, bf16_random, make_routing, to_dev_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    assert _t.cuda.is_available()
    return _t


def _check_normal(R, E, xs, idxs, ws, recv, comb, n_worst=0):
    """recv[d] = (recv_x, recv_topk_idx, recv_topk_w, handle); comb[s] = (x, w)."""
    in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
    out, heads = O.dispatch(xs, in_ranks, idxs, ws, E)
    for d in range(R):
        rx, ti, tw, h = recv[d]
        n = out[d]["recv_x"].shape[0]
        if n_worst:
            assert rx.shape[0] == n_worst and ti.shape[0] == n_worst
            assert (ti[n:].cpu().numpy() == -1).all(), "rows past the real count must carry no expert"
        assert np.array_equal(bf16_bits(rx[:n]), out[d]["recv_x"]), d
        assert np.array_equal(ti[:n].cpu().numpy(), out[d]["recv_topk_idx"]), d
        assert np.array_equal(tw[:n].cpu().numpy(), out[d]["recv_topk_weights"]), d
        assert np.array_equal(h[3][:n].cpu().numpy(), out[d]["recv_src_idx"]), d
    ref = O.combine([o["recv_x"] for o in out], in_ranks, heads, out[0]["rank_prefix_matrix"],
                    [o["recv_topk_weights"] for o in out])
    for s in range(R):
        assert np.array_equal(bf16_bits(comb[s][0]), ref[s][0]), s
        assert np.array_equal(comb[s][1].cpu().numpy(), ref[s][1]), s


def test_num_worst_tokens_graph_replay(torch):
    """Buffer (one rank): layout -> dispatch(num_worst_tokens) -> combine captured in
    one CUDA graph and replayed on new inputs copied into the static buffers;
    eager calls before and after the replays stay in step (device-resident epochs)."""
    from paper_2512_19849_b200 import Buffer, nvl_bytes_hint
    T, H, E, k = 1024, 2048, 64, 8
    buf = Buffer(None, nvl_bytes_hint(T, H, 1, k))
    g = np.random.default_rng(3)

    def inputs():
        idx, w = make_routing(g, T, E, k, mask_frac=0.05)
        return bf16_random(g, (T, H)), idx, w

    sx = torch.empty((T, H), dtype=torch.bfloat16, device="cuda")
    si = torch.empty((T, k), dtype=torch.int64, device="cuda")
    sw = torch.empty((T, k), dtype=torch.float32, device="cuda")

    def load(x, idx, w):
        sx.copy_(to_dev_bf16(x))
        si.copy_(torch.from_numpy(idx))
        sw.copy_(torch.from_numpy(w))

    def step(n_worst):
        per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(si, E)
        rx, rti, rtw, lst, handle, _ = buf.dispatch(sx, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank,
                                                    num_tokens_per_expert=per_exp, topk_idx=si, topk_weights=sw,
                                                    num_worst_tokens=n_worst)
        out, out_w, _ = buf.combine(rx, handle, topk_weights=rtw)
        return rx, rti, rtw, lst, handle, out, out_w

    x, idx, w = inputs()  # eager, no worst-case sizing
    load(x, idx, w)
    rx, rti, rtw, lst, h, out, out_w = step(0)
    torch.cuda.synchronize()
    _check_normal(1, E, [x], [idx], [w], [(rx, rti, rtw, h)], [(out, out_w)])
    assert lst == np.bincount(idx[idx >= 0], minlength=E).tolist()
    del rx, rti, rtw, h, out, out_w

    graph = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        step(T)  # warm-up on the capture stream
        with torch.cuda.graph(graph, stream=st):
            rx, rti, rtw, lst, h, out, out_w = step(T)
    torch.cuda.current_stream().wait_stream(st)
    assert lst == []
    for _ in range(3):
        x, idx, w = inputs()
        load(x, idx, w)
        graph.replay()
        torch.cuda.synchronize()
        _check_normal(1, E, [x], [idx], [w], [(rx, rti, rtw, h)], [(out, out_w)], n_worst=T)
    del rx, rti, rtw, h, out, out_w, graph
    x, idx, w = inputs()  # eager again after the replays
    load(x, idx, w)
    rx, rti, rtw, lst, h, out, out_w = step(0)
    torch.cuda.synchronize()
    _check_normal(1, E, [x], [idx], [w], [(rx, rti, rtw, h)], [(out, out_w)])
    buf._g.check_device_error()
    del rx, rti, rtw, h, out, out_w
    buf.destroy()


def test_num_worst_tokens_local_group(torch):
    """R = 4 emulated ranks: worst-case sized outputs (R*T rows), then a normal call."""
    from paper_2512_19849_b200 import LocalGroup, nvl_bytes_hint
    R, T, H, E, k = 4, 300, 1024, 32, 4
    grp = LocalGroup(R, nvl_bytes_hint(T, H, R, k, 2), num_recv_slots=2)
    g = np.random.default_rng(9)
    for n_worst in (R * T, 0, R * T):
        xs, idxs, ws = [], [], []
        for _ in range(R):
            idx, w = make_routing(g, T, E, k)
            xs.append(bf16_random(g, (T, H)))
            idxs.append(idx)
            ws.append(w)
        topk = [torch.from_numpy(i).cuda() for i in idxs]
        lay = grp.get_dispatch_layout(topk, E)
        res = grp.dispatch([to_dev_bf16(x) for x in xs], [l[3] for l in lay], [l[2] for l in lay], topk,
                           [torch.from_numpy(w).cuda() for w in ws], num_worst_tokens=n_worst)
        comb = grp.combine([r[0] for r in res], [r[4] for r in res], [r[2] for r in res])
        torch.cuda.synchronize()
        grp.check_device_error()
        _check_normal(R, E, xs, idxs, ws, [(r[0], r[1], r[2], r[4]) for r in res], comb, n_worst=n_worst)
        if n_worst:
            assert all(r[3] == [] for r in res)
        del res, comb
    grp.destroy()


def test_num_worst_tokens_too_small_reports(torch):
    from paper_2512_19849_b200 import Buffer, ConfigError, nvl_bytes_hint
    T, H, E, k = 256, 1024, 16, 4
    buf = Buffer(None, nvl_bytes_hint(T, H, 1, k))
    g = np.random.default_rng(1)
    idx, w = make_routing(g, T, E, k)
    x = to_dev_bf16(bf16_random(g, (T, H)))
    ti, tw = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
    per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(ti, E)
    buf.dispatch(x, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank, num_tokens_per_expert=per_exp,
                 topk_idx=ti, topk_weights=tw, num_worst_tokens=T // 2)
    torch.cuda.synchronize()
    with pytest.raises(ConfigError):
        buf._g.check_device_error()
    with pytest.raises(ConfigError):  # larger than the receive slot
        buf.dispatch(x, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank, num_tokens_per_expert=per_exp,
                     topk_idx=ti, topk_weights=tw, num_worst_tokens=1 << 30)
    buf.destroy()


def test_comm_stream_async_finish(torch):
    """previous_event / async_finish / allocate_on_comm_stream: the ops run on
    Buffer.get_comm_stream(); the caller syncs through the returned EventOverlap."""
    from paper_2512_19849_b200 import Buffer, EventOverlap, nvl_bytes_hint
    T, H, E, k = 512, 2048, 32, 8
    buf = Buffer(None, nvl_bytes_hint(T, H, 1, k))
    comm = buf.get_comm_stream()
    assert comm != torch.cuda.current_stream()
    g = np.random.default_rng(4)
    idx, w = make_routing(g, T, E, k)
    xb = bf16_random(g, (T, H))
    x = to_dev_bf16(xb)
    ti, tw = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
    ev0 = torch.cuda.Event()
    ev0.record()
    per_rank, _, per_exp, in_rank, ev1 = buf.get_dispatch_layout(ti, E, previous_event=EventOverlap(ev0),
                                                                 async_finish=True, allocate_on_comm_stream=True)
    assert ev1.event is not None
    rx, rti, rtw, lst, handle, ev2 = buf.dispatch(x, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank,
                                                  num_tokens_per_expert=per_exp, topk_idx=ti, topk_weights=tw,
                                                  previous_event=ev1, async_finish=True)
    out, out_w, ev3 = buf.combine(rx, handle, topk_weights=rtw, previous_event=ev2, async_finish=True)
    ev3.current_stream_wait()
    torch.cuda.current_stream().synchronize()
    _check_normal(1, E, [xb], [idx], [w], [(rx, rti, rtw, handle)], [(out, out_w)])
    # async_finish=False with a previous event: the compute stream waits for the comm stream
    out2, _, ev4 = buf.combine(rx, handle, previous_event=EventOverlap(ev0))
    assert ev4.event is None
    assert torch.equal(out2, out)
    buf.destroy()


def test_zero_copy_ll_combine_buffer(torch):
    """get_next_low_latency_combine_buffer + low_latency_combine(zero_copy=True)."""
    from paper_2512_19849_b200 import Buffer
    T, H, E, k = 64, 2048, 32, 4
    buf = Buffer(None, 1 << 20, Buffer.get_low_latency_rdma_size_hint(T, H, 1, E, num_topk=k), low_latency_mode=True)
    g = np.random.default_rng(6)
    idx, w = make_routing(g, T, E, k)
    xb = bf16_random(g, (T, H))
    ti, tw = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
    recv, count, handle, _, _ = buf.low_latency_dispatch(to_dev_bf16(xb), ti, T, E, use_fp8=False)
    y = buf.get_next_low_latency_combine_buffer(handle)
    assert tuple(y.shape) == (E, T, H)
    yb = bf16_random(g, tuple(y.shape))
    y.copy_(to_dev_bf16(yb))
    out, _, _ = buf.low_latency_combine(y, ti, tw, handle, zero_copy=True)
    torch.cuda.synchronize()
    o, _ = O.ll_dispatch([xb], [idx], E, T, use_fp8=False)
    ref = O.ll_combine([[yb[le, : o[0][le]["count"]] for le in range(E)]], [idx], [w], E)
    assert np.array_equal(bf16_bits(out), ref[0])
    assert buf.get_next_low_latency_combine_buffer(handle) is not y  # double-buffered
    buf.destroy()
