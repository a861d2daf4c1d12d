"""Real multi-GPU parity: one process per GPU, CUDA-IPC peer mappings, NVLink
stores.  Each rank checks its own outputs against the oracle computed from the
seeded inputs of every rank.  Skipped with < 2 GPUs (run via gpurun --gpus 2|4)."""
import os
import socket
import traceback

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(R, T, H, E, k, seed):
    from tests.helpers import bf16_random, make_routing
    xs, idxs, ws = [], [], []
    for r in range(R):
        g = np.random.default_rng(seed * 100 + r)
        idx, w = make_routing(g, T[r] if isinstance(T, list) else T, E, k)
        xs.append(bf16_random(g, (len(idx), H)))
        idxs.append(idx)
        ws.append(w)
    return xs, idxs, ws


def _worker(rank, world, port, results):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), EPB_TIMEOUT_S="20")
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2512_19849_b200 as epb
        from oracle import ep as O
        from tests.helpers import bf16_bits, bf16_random, to_dev_bf16, u8_bits
        R = world
        # ---- normal mode ----------------------------------------------------------
        Ts = [700 + 97 * r for r in range(R)]
        H, E, k = 7168, 64, 8
        xs, idxs, ws = _inputs(R, Ts, H, E, k, seed=1)
        topk = torch.from_numpy(idxs[rank]).cuda()
        w = torch.from_numpy(ws[rank]).cuda()
        # kernels' NVLink stores / the CPU proxy's WRITE+ATOMIC commands / bounded chunked rings
        for ht in ("nvlink", "proxy", "ring"):
            nvl = (epb.ring_nvl_bytes(H, R, k, 16, 64) if ht == "ring"
                   else epb.nvl_bytes_hint(max(Ts), H, R, k, ht_proxy=ht == "proxy"))
            buf = epb.Buffer(dist.group.WORLD, nvl, 0, fifo_channels=4, ht_transport=ht, ring_lanes=16)
            for it in range(3):  # repeat: exercises both parities / epochs and slot reuse
                per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(topk, E)
                recv_x, rti, rtw, lst, handle, _ = buf.dispatch(
                    to_dev_bf16(xs[rank]), num_tokens_per_rank=per_rank, is_token_in_rank=in_rank,
                    num_tokens_per_expert=per_exp, topk_idx=topk, topk_weights=w)
                in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
                out, heads = O.dispatch(xs, in_ranks, idxs, ws, E)
                o = out[rank]
                assert np.array_equal(bf16_bits(recv_x), o["recv_x"]), "recv_x"
                assert np.array_equal(rti.cpu().numpy(), o["recv_topk_idx"]), "recv_topk_idx"
                assert np.array_equal(rtw.cpu().numpy(), o["recv_topk_weights"]), "recv_topk_weights"
                assert lst == o["num_recv_per_expert"], "per expert"
                g = np.random.default_rng(50 + it)
                ys = [bf16_random(g, oo["recv_x"].shape) for oo in out]
                comb, comb_w, _ = buf.combine(to_dev_bf16(ys[rank]), handle, topk_weights=rtw)
                ref = O.combine(ys, in_ranks, heads, out[0]["rank_prefix_matrix"],
                                [oo["recv_topk_weights"] for oo in out])
                assert np.array_equal(bf16_bits(comb), ref[rank][0]), "combine"
                assert np.array_equal(comb_w.cpu().numpy(), ref[rank][1]), "combine weights"
            buf.destroy()
        # ---- low latency, both transports ------------------------------------------
        Tm, H2, E2, k2 = 128, 7168, 32 * R, 8
        xs2, idx2, w2 = _inputs(R, Tm, H2, E2, k2, seed=2)
        for transport in ("nvlink", "proxy"):
            ll_bytes = epb.Buffer.get_low_latency_rdma_size_hint(Tm, H2, R, E2, num_topk=k2)
            b2 = epb.Buffer(dist.group.WORLD, 1 << 20, ll_bytes, low_latency_mode=True, fifo_channels=8,
                            proxy_threads=4, ll_transport=transport)
            L = E2 // R
            for it in range(3):
                recv, count, handle, _, _ = b2.low_latency_dispatch(
                    to_dev_bf16(xs2[rank]), torch.from_numpy(idx2[rank]).cuda(), Tm, E2, use_fp8=True)
                o2, _ = O.ll_dispatch(xs2, idx2, E2, Tm, use_fp8=True)
                q = u8_bits(recv[0])
                sc = recv[1].cpu().numpy()
                cnt = count.cpu().numpy()
                for le in range(L):
                    n = o2[rank][le]["count"]
                    assert cnt[le] == n, f"{transport} count"
                    if n:
                        assert np.array_equal(q[le, :n], o2[rank][le]["x"]), f"{transport} fp8 rows"
                        assert np.array_equal(sc[le, :n], o2[rank][le]["scales"]), f"{transport} scales"
                g = np.random.default_rng(70 + it)
                ys2 = [bf16_random(g, (L, R * Tm, H2)) for _ in range(R)]
                comb, _, _ = b2.low_latency_combine(to_dev_bf16(ys2[rank]), torch.from_numpy(idx2[rank]).cuda(),
                                                    torch.from_numpy(w2[rank]).cuda(), handle)
                ref = O.ll_combine([[ys2[d][le, : o2[d][le]["count"]] for le in range(L)] for d in range(R)],
                                   idx2, w2, E2)
                assert np.array_equal(bf16_bits(comb), ref[rank]), f"{transport} LL combine"
            if transport == "proxy":
                # Barrier TransferCmd: no rank's barrier completes before the last
                # rank entered; ranks enter 0.25 s apart
                import time
                for rep in range(2):
                    dist.barrier()
                    time.sleep(0.25 * ((rank + rep) % R))
                    t_in = time.time()
                    b2.proxy_barrier(channel=rep)
                    torch.cuda.synchronize()
                    t_out = time.time()
                    ts = [None] * R
                    dist.all_gather_object(ts, (t_in, t_out))
                    assert min(o for _, o in ts) >= max(i for i, _ in ts) - 0.002, f"proxy barrier released early {ts}"
                b2.proxy_barrier(same_rail=True)  # no rail peers on one node: completes at once
                torch.cuda.synchronize()
            b2.destroy()
        dist.barrier()
        dist.destroy_process_group()
        results.put((rank, "ok"))
    except Exception:
        results.put((rank, traceback.format_exc()))


def test_multigpu_parity():
    import torch
    import torch.multiprocessing as mp
    world = min(4, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, msg = q.get(timeout=600)
        res[r] = msg
    for p in procs:
        p.join(timeout=60)
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad, "\n".join(f"rank {r}:\n{m}" for r, m in bad.items())
