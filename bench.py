"""Benchmark of the EP dispatch/combine hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 runs in-process; N > 1 is launched by the driver under torchrun (one
process per GPU, NCCL only for the start/stop barrier and the max-over-ranks
reduction of the timings; the data path itself uses no collective).

Workload (BASELINE.json configs[1]): DeepSeek-V3 normal mode, 4096 tokens per
rank, hidden 7168, 256 experts, top-8, bf16 dispatch / bf16 combine, EP = N.
A step = get_dispatch_layout -> dispatch -> combine through the public Buffer
API, on synthetic seeded inputs already resident in HBM.  Four input sets
rotate so every step's inputs (4 x 58.7 MB) were evicted from the 126 MB L2.

value = payload bytes moved per step by all ranks (dispatch rows + combine
rows, every (token, destination-rank) row counted once per direction, local
rows included) / step time, in GB/s.  `roofline` describes the dominant
kernel (HBM-bound at EP=1, NVLink-bound at EP>1).
`e2e` repeats the step from pinned host buffers (H2D of x/topk/weights, D2H of
the combined output) through the same API.  `ll` reports the low-latency
128-token FP8 dispatch + bf16 combine in microseconds (direct NVLink stores
and the GPU->CPU FIFO proxy transport).  `cpu_baseline` times the oracle port
on the box's host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context (see the package __init__)

import numpy as np  # noqa: E402

T_PER_RANK, HIDDEN, EXPERTS, TOPK = 4096, 7168, 256, 8
LL_TOKENS = 128
NSLOTS = 9  # receive slots: the captured step graphs (4 + 3) + eager + the scratch slot
ROW = HIDDEN * 2
WORKLOAD = "DeepSeek-V3 normal mode: 4096 tok/rank, hidden 7168, 256 experts, top-8, bf16 dispatch + bf16 combine"
METRIC = "dispatch/combine GB/s per GPU at 1/2/4/8 B200 (+ LL µs) vs NVLink roofline"
NVLINK_PEAK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); no NVLink entry in MEASURED_PEAKS


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def _sm_hz(index: int) -> float:
    """SM clock in Hz (NVML max clock; the B200 boost clock if NVML is absent)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        return 1e6 * pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(index), pynvml.NVML_CLOCK_SM)
    except Exception:
        return 1.965e9


class Clocks:
    """SM clock / throttle-reason sampler (NVML, every ~2 ms) running during the
    timed region — the same counters `nvidia-smi --query-gpu=clocks.sm,...,
    clocks_event_reasons.*` reports, at a rate that fits millisecond regions."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.h = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            reasons = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, reasons))

    def _run(self):
        while not self.stop.is_set():
            self._sample()
            time.sleep(0.002)

    def __exit__(self, *exc):
        if self.h is not None:
            self.stop.set()
            self.t.join(timeout=2)
            self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for _, r in self.samples for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(self.samples), "source": "NVML during the timed region"}


class NvlinkGpm:
    """NVLink bytes from NVML GPM (GPU Performance Monitoring) samples: the
    device's total NVLink TX / RX bandwidth between two samples, times the
    interval (nvidia-smi's nvlink throughput counters read N/A on this pool)."""

    def __init__(self, index: int):
        self.ok, self.source = False, "unavailable"
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            if not nv.nvmlGpmQueryDeviceSupport(self.h).isSupportedDevice:
                self.source = "GPM not supported"
                return
            self.s1, self.s2 = nv.nvmlGpmSampleAlloc(), nv.nvmlGpmSampleAlloc()
            self.ok, self.source = True, "NVML GPM NVLINK_TOTAL_{TX,RX}_PER_SEC (MiB/s) x interval"
        except Exception as exc:  # noqa: BLE001
            self.source = f"unavailable: {type(exc).__name__}: {exc}"[:120]

    def start(self):
        if self.ok:
            try:
                self.nv.nvmlGpmSampleGet(self.h, self.s1)
            except Exception as exc:  # noqa: BLE001  (e.g. GPM not permitted in this container)
                self.ok, self.source = False, f"unavailable: nvmlGpmSampleGet: {exc}"[:120]
            self.t0 = time.perf_counter()

    def stop(self):
        if not self.ok:
            return None, None
        nv = self.nv
        try:
            nv.nvmlGpmSampleGet(self.h, self.s2)
        except Exception as exc:  # noqa: BLE001
            self.ok, self.source = False, f"unavailable: nvmlGpmSampleGet: {exc}"[:120]
            return None, None
        dt = time.perf_counter() - self.t0
        mg = nv.c_nvmlGpmMetricsGet_t()
        mg.version = nv.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 2
        mg.sample1, mg.sample2 = self.s1, self.s2
        mg.metrics[0].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
        mg.metrics[1].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
        try:
            nv.nvmlGpmMetricsGet(mg)
        except Exception:  # noqa: BLE001
            return None, None
        if mg.metrics[0].nvmlReturn or mg.metrics[1].nvmlReturn:
            return None, None
        return mg.metrics[0].value * (1 << 20) * dt, mg.metrics[1].value * (1 << 20) * dt


# ----------------------------------------------------------------------------------
# CPU reference arm (the oracle port; /root/reference does not exist on the GPU box)
# ----------------------------------------------------------------------------------
def _cpu_inputs(rank: int, T: int):
    from tests.helpers import bf16_random, make_routing
    g = np.random.default_rng(1000 + rank)
    idx, w = make_routing(g, T, EXPERTS, TOPK)
    x = bf16_random(g, (T, HIDDEN))
    return x, idx, w


def _cpu_step(x, idx, w, world, threads):
    """Oracle layout -> dispatch -> combine for one rank's tokens at EP=world (the
    local view: rows to every destination, and the same rows combined back)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import ep as O
    T = x.shape[0]
    chunks = np.array_split(np.arange(T), threads)

    def part(tok):
        xs = x[tok]
        in_rank = O.get_dispatch_layout(idx[tok], EXPERTS, world)[2]
        out, heads = O.dispatch([xs] + [xs[:0]] * (world - 1), [in_rank] + [in_rank[:0]] * (world - 1))
        comb = O.combine([o["recv_x"] for o in out], [in_rank] + [in_rank[:0]] * (world - 1), heads,
                         out[0]["rank_prefix_matrix"])
        return int(in_rank.sum()), comb[0][0]
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(part, chunks))
    rows = sum(r[0] for r in res)
    return rows


def cpu_baseline(world: int, budget_s: float = 12.0, threads: int = 1):
    x, idx, w = _cpu_inputs(0, T_PER_RANK)
    _cpu_step(x, idx, w, world, threads)  # warm
    t0 = time.perf_counter()
    n, rows = 0, 0
    while time.perf_counter() - t0 < budget_s or n == 0:
        rows += _cpu_step(x, idx, w, world, threads)
        n += 1
    dt = time.perf_counter() - t0
    gbs = 2 * rows * ROW / dt / 1e9
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{n} full steps (layout+dispatch+combine of 4096x7168 bf16 tokens, EP={world} local view) "
                      f"in {dt:.1f} s with the numpy oracle"}


def _config_dict(world: int) -> dict:
    """The workload description both arms print (identical dicts: same_config)."""
    return {"workload": WORKLOAD, "ep": world, "tokens_per_rank": T_PER_RANK, "hidden": HIDDEN,
            "experts": EXPERTS, "topk": TOPK, "parallelism": f"ep{world}"}


def ref_sample_tokens(world: int) -> int:
    """Tokens per simulated rank in one reference-arm step: the full 4096 at EP=1,
    4096/EP^2 beyond, so a step's message count stays near the EP=1 one and the
    whole --steps/--warmup run ends within a few minutes."""
    return T_PER_RANK if world == 1 else max(32, T_PER_RANK // (world * world))


def run_reference(args):
    """The reference's own CPU implementation of the path (oracle/refpipe.py):
    epsim's pack_fields -> SPSC ring (2 threads) -> unpack_fields + imm encode ->
    apply_deliveries for the HT dispatch of every simulated rank, then the
    oracle port's canonical combine (the reference has no combine code)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ep as O
    from oracle import refpipe
    from tests.helpers import bf16_random, make_routing
    world = args.gpus
    Ts = ref_sample_tokens(world)
    xs, in_ranks = [], []
    for r in range(world):
        g = np.random.default_rng(1000 + r)
        idx, _ = make_routing(g, Ts, EXPERTS, TOPK)
        xs.append(bf16_random(g, (Ts, HIDDEN)))
        in_ranks.append(O.get_dispatch_layout(idx, EXPERTS, world)[2])
    dt, step_bytes, backend, cores = refpipe.time_steps(xs, in_ranks, args.steps, args.warmup)
    gbs = step_bytes / dt / 1e9
    sample = (f"{world} simulated rank(s) x {Ts} tokens (of {T_PER_RANK}) per step; epsim ({backend}) pack_fields -> "
              f"SPSC ring cap {refpipe.RING_CAP} -> unpack_fields + encode_ht_batch -> 50%-reordered "
              f"apply_deliveries (HT, {refpipe.NCH} channels, 32-token chunks; single-threaded as shipped), then "
              f"the numpy oracle's canonical combine on {cores} threads (the reference has no combine)")
    line = {"impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded routing, N(0,1) bf16 tokens)", "config": _config_dict(world),
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                             "sample": sample, "host_cores": len(os.sched_getaffinity(0))},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    group = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        group = dist.group.WORLD
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)

    import paper_2512_19849_b200 as epb
    from tests import verify

    R = world
    dev = torch.device("cuda", local_rank)
    nvl = epb.nvl_bytes_hint(T_PER_RANK, HIDDEN, R, TOPK, NSLOTS)
    ll_bytes = epb.Buffer.get_low_latency_rdma_size_hint(LL_TOKENS, HIDDEN, R, EXPERTS, num_topk=TOPK)
    buf = epb.Buffer(group, nvl, ll_bytes, low_latency_mode=True, num_recv_slots=NSLOTS, fifo_channels=16,
                     fifo_capacity=1024, ll_transport="nvlink")

    # rotating input sets (4 x 58.7 MB > 126 MB L2); seeded so any rank can
    # regenerate any other rank's set (oracle verification, tests/verify.py)
    NSETS = 4
    sets = []

    def head_inputs(r, i=0):
        idx, w = verify.routing(10_000 * r + i, T_PER_RANK, EXPERTS, TOPK)
        return verify.seeded_x(torch, 10_000 * r + i, T_PER_RANK, HIDDEN, dev), idx, w

    for i in range(NSETS):
        x, idx, w = head_inputs(rank, i)
        sets.append((x, torch.from_numpy(idx).to(dev), torch.from_numpy(w).to(dev)))
    # payload rows this rank moves per step (dispatch rows = combine rows)
    rows, remote_rows = [], []
    for x, idx, w in sets:
        m = torch.zeros(T_PER_RANK, R, dtype=torch.bool, device=dev)
        m.scatter_(1, idx // (EXPERTS // R), True)  # routing has no masked entries
        rows.append(int(m.sum()))
        m[:, rank] = False
        remote_rows.append(int(m.sum()))

    def step(i):
        x, idx, w = sets[i % NSETS]
        per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(idx, EXPERTS)
        recv_x, rti, rtw, _, handle, _ = buf.dispatch(x, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank,
                                                      num_tokens_per_expert=per_exp, topk_idx=idx, topk_weights=w)
        out, out_w, _ = buf.combine(recv_x, handle, topk_weights=rtw)
        return out

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    for i in range(max(3, args.warmup)):
        step(i)
    barrier()
    # one step of set 0 checked against the oracle (untimed)
    verified = {}
    verified["headline"] = _verify(lambda: _verify_normal_step(buf, sets[0], lambda r: head_inputs(r, 0), rank, R,
                                                               EXPERTS, None))
    barrier()

    # ---- CUDA-graph steps -----------------------------------------------------------
    # num_worst_tokens = R*T (DeepEP's worst-case sizing): the dispatch needs no
    # host sync, so layout -> dispatch -> combine of one input set is captured
    # as one graph; one graph per rotating set (its inputs are the set's static
    # tensors).  Replays are the serving loop: every replay does the step's full
    # work (the kernels move only the real rows).
    n_worst = R * T_PER_RANK
    cap_stream = torch.cuda.Stream(device=dev)

    def graph_step(i, ev=None):
        x, idx, w = sets[i % NSETS]
        if ev:
            ev[0].record()
        per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(idx, EXPERTS)
        if ev:
            ev[1].record()
        recv_x, rti, rtw, _, handle, _ = buf.dispatch(x, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank,
                                                      num_tokens_per_expert=per_exp, topk_idx=idx, topk_weights=w,
                                                      num_worst_tokens=n_worst)
        if ev:
            ev[2].record()
        out, out_w, _ = buf.combine(recv_x, handle, topk_weights=rtw)
        if ev:
            ev[3].record()
        return out, (per_rank, per_exp, in_rank, recv_x, rti, rtw, handle, out_w)

    def capture(with_events: bool, chains=None):
        """One graph per input set (chains=None), or one graph per entry of
        chains: a sequence of consecutive steps (set i, i+1, ...) in one graph,
        so back-to-back steps need one graph launch per chain."""
        graphs = []
        cap_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap_stream):
            for i in range(NSETS):  # warm-up on the capture stream (every rank runs it)
                graph_step(i)
            cap_stream.synchronize()
            if world > 1:
                dist.barrier()
            for seq in (chains or [[i] for i in range(NSETS)]):
                g = torch.cuda.CUDAGraph()
                ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)] if with_events else None
                outs, keeps = [], []
                with torch.cuda.graph(g, stream=cap_stream):
                    for i in seq:
                        out, keep = graph_step(i, ev)
                        outs.append(out)
                        keeps.append(keep)
                graphs.append((g, outs[0] if len(seq) == 1 else outs, keeps[0] if len(seq) == 1 else keeps, ev))
        torch.cuda.current_stream().wait_stream(cap_stream)
        barrier()
        return graphs

    graphs = capture(False)
    for i in range(max(3, args.warmup)):
        graphs[i % NSETS][0].replay()
    barrier()
    verified["graph"] = _verify(lambda: _verify_graph_step(graphs[0], sets[0], lambda r: head_inputs(r, 0), rank, R,
                                                           EXPERTS))
    barrier()

    # ---- timed region (device events around the K steps) --------------------------------
    # the K steps replay as graphs of NSETS consecutive steps (one graph launch per
    # 4 steps) plus one graph for the K mod NSETS remaining steps
    del graphs
    barrier()
    n_chain, rem = divmod(args.steps, NSETS)
    chains = [list(range(NSETS))] + ([list(range(rem))] if rem else [])
    cgraphs = capture(False, chains)
    for _ in range(2):
        cgraphs[0][0].replay()
    barrier()
    clocks = Clocks(local_rank)
    with clocks:
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(n_chain):
            cgraphs[0][0].replay()
        if rem:
            cgraphs[1][0].replay()
        ev1.record()
        barrier()
    ms_local = ev0.elapsed_time(ev1)
    del cgraphs
    barrier()
    ms = max_over_ranks(ms_local)
    my_rows = sum(rows[i % NSETS] for i in range(args.steps))
    my_remote = sum(remote_rows[i % NSETS] for i in range(args.steps))
    job_bytes = sum_over_ranks(2.0 * my_rows * ROW)
    value = job_bytes / (ms / 1e3) / 1e9
    ms_per_step = ms / args.steps
    launches_per_step = 3  # layout, dispatch (count exchange fused), combine

    # the same steps eager (host-launched, counts read back by the host every step)
    for i in range(3):
        step(i)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        step(i)
    e1.record()
    barrier()
    ms_eager = max_over_ranks(e0.elapsed_time(e1))
    eager = {"value": round(job_bytes / (ms_eager / 1e3) / 1e9, 3), "ms_per_step": round(ms_eager / args.steps, 4),
             "mode": "eager host launches; the host waits for the receive counts each dispatch"}
    barrier()

    # per-kernel device times: one graph per op kind, replayed back to back (the
    # layout / dispatch outputs they read are fixed), CUDA events around K
    # replays on the replaying stream; avg launch = elapsed / K.  The same loops,
    # run longer, are bracketed by NVML GPM samples (NVLink TX/RX bytes, N > 1).
    kgraphs = {}
    with torch.cuda.stream(cap_stream):
        cap_stream.wait_stream(torch.cuda.current_stream())
        fixed = []
        for i in range(NSETS):
            x, idx, w = sets[i]
            pr, _, pe, ir, _ = buf.get_dispatch_layout(idx, EXPERTS)
            fixed.append((x, idx, w, pr, pe, ir))
        rx0, _, rtw0, _, h0, _ = buf.dispatch(sets[0][0], num_tokens_per_rank=fixed[0][3], is_token_in_rank=fixed[0][5],
                                              num_tokens_per_expert=fixed[0][4], topk_idx=sets[0][1],
                                              topk_weights=sets[0][2], num_worst_tokens=n_worst)
        buf.combine(rx0, h0, topk_weights=rtw0)
        cap_stream.synchronize()
        if world > 1:
            dist.barrier()
        for kind in ("layout", "dispatch"):
            gl = []
            for i in range(NSETS):
                g = torch.cuda.CUDAGraph()
                x, idx, w, pr, pe, ir = fixed[i]
                with torch.cuda.graph(g, stream=cap_stream):
                    if kind == "layout":
                        keep = buf.get_dispatch_layout(idx, EXPERTS)
                    else:
                        keep = buf.dispatch(x, num_tokens_per_rank=pr, is_token_in_rank=ir, num_tokens_per_expert=pe,
                                            topk_idx=idx, topk_weights=w, num_worst_tokens=n_worst)
                gl.append((g, keep))
            kgraphs[kind] = gl
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap_stream):
            keep = buf.combine(rx0, h0, topk_weights=rtw0)
        kgraphs["combine"] = [(g, keep)]
    torch.cuda.current_stream().wait_stream(cap_stream)
    barrier()

    def kernel_loop(kind, n):
        gl = kgraphs[kind]
        for j in range(n):
            gl[j % len(gl)][0].replay()

    per_kernel = {}
    for kind in ("layout", "dispatch", "combine"):
        kernel_loop(kind, 3)
        barrier()
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record()
        kernel_loop(kind, args.steps)
        k1.record()
        barrier()
        per_kernel[kind] = [max_over_ranks(k0.elapsed_time(k1)) / args.steps]
    nvlink = None
    if R > 1:
        gpm = NvlinkGpm(local_rank)
        nvlink = {"source": gpm.source}
        for kind in ("dispatch", "combine"):
            reps = max(200, int(0.25 / max(1e-6, per_kernel[kind][0] / 1e3)))  # >= 0.25 s per GPM interval
            barrier()
            gpm.start()
            kernel_loop(kind, reps)
            torch.cuda.synchronize()
            tx, rx = gpm.stop()
            barrier()
            if tx is not None:
                nvlink[kind] = {"tx_bytes_per_launch": int(tx / reps), "rx_bytes_per_launch": int(rx / reps),
                                "launches": reps}
    del kgraphs
    barrier()

    # ---- SM budget (the same SMs per GPU as DeepEP) -------------------
    # dispatch / combine as one-kernel graphs with Config(num_sms=n): n blocks
    # (channels) for the dispatch, n blocks for the combine; the rest of the GPU
    # stays free for the caller's compute.
    sm_budget = {}
    if not args.no_configs:
        x0, idx0, w0, pr0, pe0, ir0 = fixed[0]
        for n_sms in (20, 24, 48):
            cfg = epb.Config(n_sms)
            with torch.cuda.stream(cap_stream):
                cap_stream.wait_stream(torch.cuda.current_stream())
                rxb, _, rtwb, _, hb, _ = buf.dispatch(x0, num_tokens_per_rank=pr0, is_token_in_rank=ir0,
                                                      num_tokens_per_expert=pe0, topk_idx=idx0, topk_weights=w0,
                                                      num_worst_tokens=n_worst, config=cfg)
                buf.combine(rxb, hb, topk_weights=rtwb, config=cfg)
                cap_stream.synchronize()
                if world > 1:
                    dist.barrier()
                gd, gc = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
                with torch.cuda.graph(gd, stream=cap_stream):
                    kd = buf.dispatch(x0, num_tokens_per_rank=pr0, is_token_in_rank=ir0, num_tokens_per_expert=pe0,
                                      topk_idx=idx0, topk_weights=w0, num_worst_tokens=n_worst, config=cfg)
                with torch.cuda.graph(gc, stream=cap_stream):
                    kc = buf.combine(rxb, hb, topk_weights=rtwb, config=cfg)
            torch.cuda.current_stream().wait_stream(cap_stream)
            barrier()
            res_ms = {}
            for name, g_ in (("dispatch", gd), ("combine", gc)):
                for _ in range(3):
                    g_.replay()
                barrier()
                k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                k0.record()
                for _ in range(args.steps):
                    g_.replay()
                k1.record()
                barrier()
                res_ms[name] = max_over_ranks(k0.elapsed_time(k1)) / args.steps
            rows0 = rows[0]
            rem0 = max_over_ranks(float(remote_rows[0]))
            ent = {"dispatch_us": round(res_ms["dispatch"] * 1e3, 2), "combine_us": round(res_ms["combine"] * 1e3, 2)}
            if R == 1:
                ent["dispatch_hbm_gbs"] = round(2.0 * rows0 * ROW / (res_ms["dispatch"] / 1e3) / 1e9, 1)
                ent["combine_hbm_gbs"] = round(2.0 * rows0 * ROW / (res_ms["combine"] / 1e3) / 1e9, 1)
            else:
                ent["dispatch_nvlink_gbs"] = round(rem0 * ROW / (res_ms["dispatch"] / 1e3) / 1e9, 1)
                ent["combine_nvlink_gbs"] = round(rem0 * ROW / (res_ms["combine"] / 1e3) / 1e9, 1)
            sm_budget[str(n_sms)] = ent
            del gd, gc, kd, kc, rxb, rtwb, hb
            barrier()
    del fixed

    # ---- roofline of the dominant kernel -------------------------------------------------
    hbm_peak, peak_kind = _peaks()
    avg = {k: statistics.mean(v) for k, v in per_kernel.items()}
    dom = max(("dispatch", "combine"), key=lambda k: avg.get(k, 0.0))
    steps_rows = my_rows / args.steps
    steps_remote = my_remote / args.steps
    if R == 1:
        algo = 2.0 * steps_rows * ROW  # read source rows + write destination rows
        bound, peak, unit = "hbm", hbm_peak, "GB/s"
    else:
        algo = steps_remote * ROW  # unique payload bytes leaving this rank over NVLink
        bound, peak, unit = "nvlink", NVLINK_PEAK_GBS, "GB/s"
    achieved = algo / (avg[dom] / 1e3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if R > 1 and nvlink and nvlink.get(dom):
        traffic = nvlink[dom]["tx_bytes_per_launch"]  # NVLink bytes this GPU sent per launch (GPM, live)
    elif tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(f"{dom}_ep{R}")
        except Exception:
            traffic = None
    roofline = {"bound": bound, "kernel": dom, "achieved": round(achieved, 2), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_kind if R == 1 else
                "B200_PROFILING.md measured peer copy (770 GB/s/direction)",
                "algorithmic_bytes_per_launch": int(algo), "avg_launch_ms": round(avg[dom], 4),
                "timing": "CUDA events around K back-to-back replays of a one-kernel graph (fixed inputs)",
                "traffic_source": ("NVML GPM NVLink TX during the kernel's replay loop" if R > 1
                                   else "ncu --set full capture (profiles/traffic.json)")}
    kernels_ms = {k: round(v, 4) for k, v in avg.items()}

    # ---- end to end from pinned host buffers ---------------------------------------------
    # Pipelined like a serving loop: step i+1's inputs go up on an H2D stream
    # into the static inputs of the graph that runs it, step i-1's result comes
    # down on a D2H stream while step i's graph replays (PCIe is full duplex).
    # Every step still moves its own inputs and result.
    egraphs = capture(False)
    hx = [s_[0].cpu().pin_memory() for s_ in sets]
    hidx = [s_[1].cpu().pin_memory() for s_ in sets]
    hw = [s_[2].cpu().pin_memory() for s_ in sets]
    hout = [torch.empty((T_PER_RANK, HIDDEN), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    comp = torch.cuda.current_stream()
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_run(n):
        done = [None] * NSETS  # compute event of the last replay of graph j (its inputs are free after it)
        outev = [None, None]   # D2H event of the last copy into host buffer b
        outsrc = [None] * NSETS  # D2H event of the last copy out of graph j's output
        up = []

        def upload(i):
            j = i % NSETS
            with torch.cuda.stream(s_h2d):
                if done[j] is not None:
                    s_h2d.wait_event(done[j])
                sets[j][0].copy_(hx[j], non_blocking=True)
                sets[j][1].copy_(hidx[j], non_blocking=True)
                sets[j][2].copy_(hw[j], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_h2d)
            up.append(ev)

        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        s_h2d.wait_event(e0)
        upload(0)
        for i in range(n):
            if i + 1 < n:
                upload(i + 1)
            j, b = i % NSETS, i % 2
            comp.wait_event(up[i])
            if outsrc[j] is not None:
                comp.wait_event(outsrc[j])  # the graph's output buffer was read out
            egraphs[j][0].replay()
            ev = torch.cuda.Event()
            ev.record(comp)
            done[j] = ev
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev)
                if outev[b] is not None:
                    s_d2h.wait_event(outev[b])
                hout[b].copy_(egraphs[j][1], non_blocking=True)
                oe = torch.cuda.Event()
                oe.record(s_d2h)
                outev[b] = oe
                outsrc[j] = oe
        for b in range(2):
            if outev[b] is not None:
                comp.wait_event(outev[b])
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(comp)
        return e0, e1

    e2e_run(3)
    barrier()
    e0, e1 = e2e_run(args.steps)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    h2d = T_PER_RANK * ROW + T_PER_RANK * TOPK * 12
    d2h = T_PER_RANK * ROW
    e2e = {"value": round(job_bytes / (e2e_ms / 1e3) / 1e9, 4), "unit": "GB/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms / args.steps, 4),
           "pipelining": "H2D of step i+1 and D2H of step i-1 overlap step i's graph replay (separate copy streams)"}
    del egraphs
    barrier()

    # ---- the other normal-mode rows of BASELINE.json (per-op device times) -------------------
    configs = {}
    if not args.no_configs:
        common = (rank, R, dev, args, barrier, max_over_ranks, group)
        for name, kw in (("dsv3_fp8_dispatch", dict(T=T_PER_RANK, H=HIDDEN, E=EXPERTS, fp8=True, buf=buf)),
                         ("dsv3_bf16_combine_push", dict(T=T_PER_RANK, H=HIDDEN, E=EXPERTS, combine_in_region=False,
                                                         buf=buf)),
                         ("qwen3_235b_zipf", dict(T=8192, H=4096, E=128, zipf=1.0)),
                         ("dsv3_bf16_ring", dict(T=T_PER_RANK, H=HIDDEN, E=EXPERTS, ht="ring")),
                         ("dsv3_bf16_ht_proxy", dict(T=T_PER_RANK, H=HIDDEN, E=EXPERTS, ht="proxy"))):
            only = os.environ.get("EPB_BENCH_CONFIGS")
            if only and name not in only.split(","):
                continue
            try:
                configs[name] = config_bench(name, *common, **kw)
            except Exception as exc:
                configs[name] = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    # ---- low-latency decode (128 tokens, FP8 dispatch + bf16 combine) ----------------------
    ll = {}
    for transport in (() if args.no_ll else ("nvlink", "proxy")):
        try:
            ll[transport] = ll_bench(buf, transport, rank, R, dev, args, barrier, max_over_ranks)
        except Exception as exc:  # keep the headline even if a transport is unavailable
            ll[transport] = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    # ---- GPU -> CPU FIFO: device-producer command rate --
    fifo = None
    if not args.no_ll:
        try:
            import ctypes as C
            from paper_2512_19849_b200._lib import check, lib
            if not buf._rank.proxy_running:
                check(lib.epb_proxy_start(buf._rank.ctx))
                buf._rank.proxy_running = True
            n_cmds, chans = 1 << 20, 8
            el = C.c_int64()
            check(lib.epb_fifo_device_bench(buf._rank.ctx, n_cmds, chans, C.byref(el),
                                            torch.cuda.current_stream().cuda_stream))
            fifo = {"mcmd_s": round(n_cmds / (el.value / 1e9) / 1e6, 2), "commands": n_cmds, "channels": chans,
                    "proxy_threads": buf._rank.cfg.proxy_threads,
                    "how": "one producer warp per channel pushes 16-byte TransferCmds in 32-slot bursts into pinned "
                           "rings; the proxy threads pop them (count-only) and publish COMPLETED; device-timed "
                           "until every command is completed"}
        except Exception as exc:  # noqa: BLE001
            fifo = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    buf._g.check_device_error()
    line = None
    if rank == 0:
        cpu = cpu_baseline(R) if (R == 1 and not args.no_cpu_baseline) else None
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": R, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded uniform top-8 routing, N(0,1) bf16 tokens)",
                "config": _config_dict(R),
                "l2": f"{NSETS} rotating input sets ({NSETS * T_PER_RANK * ROW / 1e6:.0f} MB > 126 MB L2)",
                "value_scope": "sum over all GPUs of the payload bytes each moves per step (dispatch + combine rows, "
                               "local rows included) / max-over-ranks step time",
                "per_gpu_gbs": round(value / R, 3),
                "verified": {"verified": all(v.get("verified") for v in verified.values()), **verified},
                "step_mode": f"CUDA graphs of {NSETS} consecutive steps (layout -> dispatch(num_worst_tokens="
                             f"{n_worst}) -> combine per step), replayed back to back",
                "eager": eager, "kernels_ms": kernels_ms, "sm_budget": sm_budget, "nvlink_hw": nvlink,
                "fifo_device_producer": fifo, "roofline": roofline, "e2e": e2e, "ll_us": ll, "configs": configs,
                "gpu_launches": launches_per_step * args.steps, "gpu_launches_scope": "per rank",
                "clocks": clocks.summary(), "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    buf.destroy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _verify(fn):
    """Run one oracle check (untimed); never let a failure take the bench line down."""
    try:
        info = fn()
        return {"verified": True, **(info or {})}
    except Exception as exc:  # noqa: BLE001
        return {"verified": False, "verify_error": f"{type(exc).__name__}: {exc}"[:300]}


def _verify_normal_step(buf, inp, inputs_fn, rank, R, E, fp8_cast, combine_copy=False):
    """layout -> dispatch -> combine (identity experts) of one input set through the
    public API, then tests/verify.py against the oracle on every rank."""
    import torch
    from tests import verify
    x, idx, w = inp
    x_in = fp8_cast(x) if fp8_cast else x
    per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(idx, E)
    recv_x, rti, rtw, lst, handle, _ = buf.dispatch(x_in, num_tokens_per_rank=per_rank, is_token_in_rank=in_rank,
                                                    num_tokens_per_expert=per_exp, topk_idx=idx, topk_weights=w)
    if fp8_cast:
        y = recv_x[0].to(torch.bfloat16)
    else:
        y = recv_x.clone() if combine_copy else recv_x
    out, out_w, _ = buf.combine(y, handle, topk_weights=rtw)
    torch.cuda.synchronize()
    buf._g.check_device_error()
    return verify.verify_normal(torch, rank, R, E, inputs_fn, (recv_x, rti, rtw, lst, handle), (out, out_w),
                                fp8_cast=fp8_cast, check_tokens=None if R == 1 else 512)


def _verify_graph_step(graph, inp, inputs_fn, rank, R, E):
    """One replay of a captured step graph (num_worst_tokens outputs) against the oracle."""
    import torch
    from tests import verify
    g, out, keep, _ = graph
    g.replay()
    torch.cuda.synchronize()
    per_rank, per_exp, in_rank, recv_x, rti, rtw, handle, out_w = keep
    n = int(handle[0][R - 1, rank])  # real receive rows (rank_prefix_matrix)
    assert (rti[n:] == -1).all(), "rows past the real count must carry no expert"
    h = tuple(t[:n] if i == 3 else t for i, t in enumerate(handle))
    return verify.verify_normal(torch, rank, R, E, inputs_fn, (recv_x[:n], rti[:n], rtw[:n], [], h), (out, out_w),
                                check_tokens=None if R == 1 else 512, check_per_expert=False)


def config_bench(name, rank, R, dev, args, barrier, max_over_ranks, group, *, T, H, E, fp8=False, zipf=0.0,
                 combine_in_region=True, buf=None, ht="nvlink"):
    """Per-op device times of the other BASELINE.json normal-mode rows
    (SURVEY.md §8(d)): FP8 dispatch of DS-V3, Qwen3-235B with Zipf routing,
    and combine on expert outputs allocated OUTSIDE the arena (push mode).
    L2 is flushed (256 MB memset) before every op pair; the times are the
    median over reps of the max over ranks, from CUDA events on the stream."""
    import torch
    import paper_2512_19849_b200 as epb
    own = buf is None
    if own and ht == "ring":  # bounded rings: 74 lanes x 64 slots per peer, whatever T is (tools/ring_sweep.py)
        buf = epb.Buffer(group, epb.ring_nvl_bytes(H, R, TOPK, 74, 64), 0, ht_transport="ring", ring_lanes=74)
    elif own:
        buf = epb.Buffer(group, epb.nvl_bytes_hint(T, H, R, TOPK, 2, ht_proxy=ht == "proxy"), 0, num_recv_slots=2,
                         fifo_channels=8 if ht == "proxy" else 0, ht_transport=ht)
    from tests import verify

    def inputs(r):
        seed = 31_000 + 97 * r + int(zipf * 10)
        idx, w = verify.routing(seed, T, E, TOPK, zipf=zipf)
        return verify.seeded_x(torch, seed, T, H, dev), idx, w

    x, idx, w = inputs(rank)
    idx_t, w_t = torch.from_numpy(idx).to(dev), torch.from_numpy(w).to(dev)
    x_in = epb.per_token_cast_to_fp8(x) if fp8 else x
    check = _verify(lambda: _verify_normal_step(buf, (x, idx_t, w_t), inputs, rank, R, E,
                                                epb.per_token_cast_to_fp8 if fp8 else None,
                                                combine_copy=not combine_in_region))
    barrier()
    row_bytes = (H + 4 * (H // 128)) if fp8 else 2 * H
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    m = torch.zeros(T, R, dtype=torch.bool, device=dev)
    m.scatter_(1, idx_t // (E // R), True)
    m[:, rank] = False
    remote = int(m.sum())
    reps = max(10, min(args.steps, 30))
    d_ms, c_ms = [], []
    try:
        out = _config_loop(buf, own, idx_t, w_t, x_in, fp8, combine_in_region, flush, remote, reps, T, H, E, zipf, ht,
                           row_bytes, R, dev, barrier, max_over_ranks, d_ms, c_ms)
        out.update(check)
        return out
    except Exception:
        if ht == "proxy":
            _proxy_diag(buf, rank)
        raise


def _proxy_diag(buf, rank):
    """stderr dump of the proxy state of one rank (FIFO ctl words, counters)."""
    import ctypes as C
    import torch
    from paper_2512_19849_b200._lib import lib
    from paper_2512_19849_b200.buffer import _SlotMemory
    rk = buf._rank
    st = (C.c_int64 * 3)()
    lib.epb_proxy_stats(rk.ctx, st)
    ctl = []
    for ch in range(rk.cfg.fifo_channels):
        q, cap = C.POINTER(C.c_int64)(), C.c_int64()
        lib.epb_fifo_ctl(rk.ctx, ch, C.byref(q), C.byref(cap))
        ctl.append((q[0], q[8], q[16]))
        if q[0]:
            from paper_2512_19849_b200 import command as cmdmod
            for i in range(q[0]):
                lo, hi = q[32 + 2 * i] & (2**64 - 1), q[33 + 2 * i] & (2**64 - 1)
                c = cmdmod.unpack(lo, hi)
                print(f"   ch{ch} #{i}: kind={c.kind} dst={c.dst_rank} so={c.src_offset} do={c.dst_offset} "
                      f"len={c.length_or_value} flags={c.flags}", file=sys.stderr, flush=True)
    off = lib.epb_debug_ht_sig_offset()
    sig = torch.as_tensor(_SlotMemory(rk.base + off, 128), device=rk.device).view(torch.int64).cpu().tolist()
    print(f"[proxy diag rank {rank}] served/copies/atomics {list(st)} ctl(tail,head,completed) {ctl} "
          f"ht_sig {sig[:8]} | {sig[8:]}", file=sys.stderr, flush=True)


def _config_loop(buf, own, idx_t, w_t, x_in, fp8, combine_in_region, flush, remote, reps, T, H, E, zipf, ht,
                 row_bytes, R, dev, barrier, max_over_ranks, d_ms, c_ms):
    import torch
    import paper_2512_19849_b200 as epb
    # device time of each launch from the extension's own events (recorded
    # around the kernel launch, not after the host's wait for the counts); an
    # L2 flush and a short spin run ahead of each op so its start event is
    # already queued when the GPU gets there
    spin = int(20e-6 * _sm_hz(torch.cuda.current_device()))
    for it in range(reps + 3):
        per_rank, _, per_exp, in_rank, _ = buf.get_dispatch_layout(idx_t, E)
        barrier()
        prof = []
        flush.zero_()
        torch.cuda._sleep(spin)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()  # ring transport: Python host path (count exchange, host sync, ring kernel)
        with epb.buffer.profiling(prof):
            recv_x, _, rtw, _, handle, _ = buf.dispatch(x_in, num_tokens_per_rank=per_rank,
                                                        is_token_in_rank=in_rank, num_tokens_per_expert=per_exp,
                                                        topk_idx=idx_t, topk_weights=w_t)
        ev[1].record()
        if fp8 or not combine_in_region:  # expert outputs live in ordinary device memory
            y = torch.empty((recv_x[0] if fp8 else recv_x).shape[0], H, dtype=torch.bfloat16, device=dev)
            y.copy_(recv_x[0].to(torch.bfloat16) if fp8 else recv_x)
        else:
            y = recv_x
        flush.zero_()
        torch.cuda._sleep(spin)
        ev[2].record()
        with epb.buffer.profiling(prof):
            buf.combine(y, handle, topk_weights=rtw)
        ev[3].record()
        barrier()
        t = dict(prof)
        if ht == "ring":
            t = {"dispatch": ev[0].elapsed_time(ev[1]), "combine": ev[2].elapsed_time(ev[3])}
        if it >= 3:
            d_ms.append(max_over_ranks(t["dispatch"]))
            c_ms.append(max_over_ranks(t["combine"]))
        del recv_x, y, handle
    buf._g.check_device_error()
    if own:
        buf.destroy()
    rem_max = max_over_ranks(float(remote))
    d, c = statistics.median(d_ms), statistics.median(c_ms)
    out = {"tokens_per_rank": T, "hidden": H, "experts": E, "topk": TOPK, "dispatch_dtype": "fp8" if fp8 else "bf16",
           "routing": f"zipf({zipf})" if zipf else "uniform",
           "transport": {"proxy": "CPU proxy (FIFO + copy engine)",
                         "ring": f"bounded chunked rings ({buf.num_nvl_bytes / 1e6:.0f} MB arena, 74 lanes x 64 "
                                 "slots per peer; worst-case slots would need "
                                 f"{epb.nvl_bytes_hint(T, H, R, TOPK, 2) / 1e6:.0f} MB)"}.get(
                             ht, "SM stores/loads over NVLink"), "dispatch_us": round(d * 1e3, 2),
           "combine_us": round(c * 1e3, 2), "combine_input": "device tensor (ring transport)" if ht == "ring"
           else ("arena view (WRITE in place)" if ht == "proxy" else "arena view (pull)")
           if y_in_region(fp8, combine_in_region)
           else "device tensor outside the arena (push)", "reps": reps}
    if R > 1:
        out["max_remote_rows"] = int(rem_max)
        out["dispatch_nvlink_gbs"] = round(rem_max * row_bytes / (d / 1e3) / 1e9, 1)
        out["combine_nvlink_gbs"] = round(rem_max * 2 * H / (c / 1e3) / 1e9, 1)
    return out


def y_in_region(fp8, combine_in_region):
    return combine_in_region and not fp8


def ll_bench(buf, transport, rank, R, dev, args, barrier, max_over_ranks):
    import torch
    from paper_2512_19849_b200._lib import check, lib
    if transport == "proxy" and not buf._rank.proxy_running:
        check(lib.epb_proxy_start(buf._rank.ctx))
        buf._rank.proxy_running = True
    buf.ll_transport = transport
    from tests import verify
    L = EXPERTS // R

    def inputs(r):
        idx, w = verify.routing(77 + r, LL_TOKENS, EXPERTS, TOPK)
        return verify.seeded_x(torch, 77 + r, LL_TOKENS, HIDDEN, dev), idx, w

    def ys(r):  # rank r's expert outputs (seeded: every rank can regenerate them)
        return verify.seeded_x(torch, 88 + r, L * R * LL_TOKENS, HIDDEN, dev).view(L, R * LL_TOKENS, HIDDEN)

    x, idx, w = inputs(rank)
    idx_t = torch.from_numpy(idx).to(dev)
    w_t = torch.from_numpy(w).to(dev)
    y = ys(rank)

    def once():
        recv, count, handle, _, _ = buf.low_latency_dispatch(x, idx_t, LL_TOKENS, EXPERTS, use_fp8=True)
        out, _, _ = buf.low_latency_combine(y, idx_t, w_t, handle)
        return out

    def disp_only():
        return buf.low_latency_dispatch(x, idx_t, LL_TOKENS, EXPERTS, use_fp8=True)[2]

    for _ in range(5):
        once()
    barrier()
    n = max(20, args.steps)

    def timed(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / reps * 1e3)

    eager_us = timed(once, n)
    out = {"tokens": LL_TOKENS, "fp8": True, "eager_step_us": round(eager_us, 2)}

    def check():
        recv, count, handle, _, _ = buf.low_latency_dispatch(x, idx_t, LL_TOKENS, EXPERTS, use_fp8=True)
        comb, _, _ = buf.low_latency_combine(y, idx_t, w_t, handle)
        torch.cuda.synchronize()
        buf._g.check_device_error()
        return verify.verify_ll(torch, rank, R, EXPERTS, LL_TOKENS, inputs, ys, recv, count, handle, comb)
    out.update(_verify(check))
    barrier()
    # decode runs dispatch+combine inside CUDA graphs (epochs are device-resident,
    # so a captured pair replays correctly); replayed back to back this is the
    # device latency of the pair, free of Python launch overhead
    try:
        handle = disp_only()
        g_pair, g_disp, g_comb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g_pair, stream=s):
                once()
            with torch.cuda.graph(g_disp, stream=s):
                disp_only()
            with torch.cuda.graph(g_comb, stream=s):
                buf.low_latency_combine(y, idx_t, w_t, handle)
        torch.cuda.current_stream().wait_stream(s)
        for g in (g_pair, g_disp, g_comb):
            g.replay()
        torch.cuda.synchronize()
        out["step_us"] = round(timed(g_pair.replay, n), 2)
        out["dispatch_us"] = round(timed(g_disp.replay, n), 2)
        out["combine_us"] = round(timed(g_comb.replay, n), 2)
        out["timing"] = "CUDA-graph replays, back to back, max over ranks"
    except Exception as exc:
        out["graph_error"] = f"{type(exc).__name__}: {exc}"[:200]
        out["step_us"] = round(eager_us, 2)
    buf._g.check_device_error()
    buf.ll_transport = "nvlink"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ll", action="store_true", help="skip the low-latency sub-benchmarks (e.g. under ncu)")
    ap.add_argument("--no-configs", action="store_true", help="skip the FP8 / push-combine / Qwen3 sub-benchmarks")
    args = ap.parse_args()
    if os.environ.get("EPB_BENCH_WATCHDOG"):  # debugging: dump every thread's stack and exit after N s
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["EPB_BENCH_WATCHDOG"]), exit=True)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
