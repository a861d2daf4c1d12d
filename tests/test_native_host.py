"""CPU tests of the C ABI (no GPU): the library loads and exports every symbol
include/epb.h declares; the host-side codecs, SPSC ring and the C++ port of
apply_deliveries reproduce the golden vectors produced by the reference."""
import re
import subprocess
import threading
import time
from pathlib import Path

import numpy as np
import pytest

from paper_2512_19849_b200 import _lib, command, imm, kernels
from paper_2512_19849_b200.errors import ChannelShutdown, ProtocolViolation
from paper_2512_19849_b200.fifo import FifoChannel
from tests.golden import toy

ROOT = Path(__file__).resolve().parents[1]
G = ROOT / "tests" / "golden"


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "epb.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(epb_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True, check=True)
    exported = {line.split()[-1] for line in nm.stdout.splitlines() if " T " in line}
    missing = declared - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"
    assert declared == set(_lib.EXPORTED)
    # every kernel in the .so is compiled for sm_100a
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode == 0:
        assert "sm_100a" in out.stdout


def test_codec_matches_reference_golden():
    d = np.load(G / "codec.npz")
    f = [d[f"f_{k}"] for k in ("kind", "dst_rank", "channel_id", "src_offset", "dst_offset", "length_or_value", "flags")]
    lo, hi = command.pack_fields(*f)
    assert np.array_equal(lo, d["lo"]) and np.array_equal(hi, d["hi"])
    back = command.unpack_fields(d["lo"], d["hi"])
    for k, v in back.items():
        assert np.array_equal(v, d[f"u_{k}"]), k
    for i in range(64):
        c = command.TransferCmd(*[int(a[i]) for a in f])
        assert command.to_bytes(c) == d["records"][i].tobytes()
        assert command.from_bytes(d["records"][i].tobytes()) == c
    kat = command.TransferCmd(0, 3, 5, 0x12345678, 0xABCDEF01, 7168, 1)
    assert command.pack(kat) == (0xF01123456781400C, 0x100001C00ABCDE)
    for h in d["bad_hi"]:
        with pytest.raises(ProtocolViolation):
            command.unpack(0, int(h))
    for bad in (dict(kind=4), dict(kind=0, dst_rank=4096), dict(kind=0, channel_id=64), dict(kind=0, flags=4),
                dict(kind=0, src_offset=1 << 32), dict(kind=0, length_or_value=-1)):
        with pytest.raises(ProtocolViolation):
            command.pack(command.TransferCmd(**bad))


def test_imm_matches_reference_golden():
    d = np.load(G / "codec.npz")
    assert np.array_equal(imm.encode_ll_batch(d["ll_k"], d["ll_c"], d["ll_o"]), d["ll_out"])
    assert np.array_equal(imm.encode_ht_batch(d["ht_k"], d["ht_c"], d["ht_s"], d["ht_o"]), d["ht_out"])
    kat = d["imm_kat"].tolist()
    assert imm.encode_ll(imm.ATOMIC, 7, 3) == kat[0]
    assert imm.encode_ht(imm.DATA, 3, 70000, 0x81) == kat[1]
    assert list(imm.decode_ht(kat[1])) == kat[2:6]
    with pytest.raises(ProtocolViolation):
        imm.ht_atomic_operand(False, 0)


def test_ring_matches_reference_golden():
    d = np.load(G / "ring.npz")
    cap = int(d["cap"])
    ctl = np.zeros(kernels.ctl_words(cap), np.int64)
    lo_out = np.zeros_like(d["lo_out"])
    hi_out = np.zeros_like(d["hi_out"])
    pushed = popped = 0
    for (op, want), r_ref, snap in zip(d["script"], d["results"], d["snaps"]):
        if op == 0:
            r = kernels.push_batch(ctl, cap, d["lo_src"], d["hi_src"], pushed, int(want), 0)
            pushed += r
        else:
            r = kernels.pop_batch(ctl, cap, lo_out, hi_out, popped, int(want), 0)
            popped += r
        assert r == r_ref
        assert np.array_equal(ctl, snap)
    assert np.array_equal(lo_out, d["lo_out"])


def _run_native_apply(regions, counters, n_used, base, mode_ht, msgs, ep, nctr, nch, pmax=8, wmax=64):
    n = len(msgs["t_del"])
    st = dict(ll_counts=np.zeros((ep, ep, nctr), np.int64), ll_px=np.zeros((ep, ep, nctr, pmax), np.int32),
              ll_pd=np.zeros((ep, ep, nctr, pmax), np.int32), ll_pn=np.zeros((ep, ep, nctr), np.int32),
              hta=np.zeros((ep, ep, nch), np.int64), htp=np.zeros((ep, ep, nch, wmax), np.int32))
    eff = [np.zeros(2 * n + 16, np.int64) for _ in range(8)]
    esc = np.zeros(max(n, 1), np.int64)
    res = kernels.apply_deliveries(regions, counters, n_used, base, mode_ht, msgs["t_del"], msgs["src"], msgs["dst"],
                                   msgs["src_off"], msgs["dst_off"], msgs["length"], msgs["op_hw"], msgs["imm"],
                                   msgs["work"], st["ll_counts"], st["ll_px"], st["ll_pd"], st["ll_pn"], st["hta"],
                                   st["htp"], *eff, esc)
    return res, np.stack([e[: res[0]] for e in eff]), st


def _kat_msgs(arr):
    keys = ("t_del", "src", "dst", "src_off", "dst_off", "length", "op_hw", "imm", "work")
    return {k: np.ascontiguousarray(arr[i]) for i, k in enumerate(keys)}


def test_native_apply_deliveries_kats():
    d = np.load(G / "deliveries_kat.npz")
    regions = np.zeros((2, 64), np.uint8)
    regions[0, :8] = np.arange(8)
    counters = np.zeros((2, 16), np.int64)
    res, eff, _ = _run_native_apply(regions, counters, 8, 0, 0, _kat_msgs(d["ll_msgs"]), 2, 16, 4)
    assert list(res) == d["ll_res"].tolist() and np.array_equal(eff, d["ll_eff"])
    assert np.array_equal(counters, d["ll_counters"]) and np.array_equal(regions, d["ll_regions"])
    regions = np.zeros((2, 64), np.uint8)
    regions[0, :8] = np.arange(10, 18)
    counters = np.zeros((2, 32), np.int64)
    res, eff, _ = _run_native_apply(regions, counters, 8, 0, 1, _kat_msgs(d["ht_msgs"]), 2, 32, 4)
    assert list(res) == d["ht_res"].tolist() and np.array_equal(eff, d["ht_eff"])
    assert np.array_equal(counters, d["ht_counters"]) and np.array_equal(regions, d["ht_regions"])


@pytest.mark.parametrize("mode", ["ht", "ll"])
def test_native_apply_deliveries_toy_dispatch(mode):
    d = np.load(G / f"{mode}_dispatch.npz")
    xs, idxs, _ = toy.make_inputs(0)
    L = toy.E // toy.EP
    if mode == "ht":
        msgs, _ = toy.ht_plan(xs, idxs)
        regions = toy.regions_init(xs, toy.EP * toy.T)
        nctr = 2 * toy.EP * toy.NCH
        counters = np.zeros((toy.EP, nctr), np.int64)
        res, eff, st = _run_native_apply(regions, counters, nctr, 0, 1, msgs, toy.EP, nctr, toy.NCH, wmax=512)
        assert np.array_equal(toy.ht_recv_blocks(regions, idxs), d["blocks"])
        assert np.array_equal(st["hta"], d["ht_applied"])
    else:
        msgs, _ = toy.ll_plan(xs, idxs)
        regions = toy.regions_init(xs, L * toy.EP * toy.T)
        counters = np.zeros((toy.EP, L), np.int64)
        res, eff, st = _run_native_apply(regions, counters, L, 0, 0, msgs, toy.EP, L, toy.NCH)
        assert np.array_equal(toy.ll_recv_blocks(regions, idxs), d["blocks"])
        assert np.array_equal(st["ll_counts"], d["ll_counts"])
    assert list(res) == d["res"].tolist()
    assert np.array_equal(eff, d["eff"])
    assert np.array_equal(counters, d["counters"])
    assert np.array_equal(np.stack([toy.digest_rows(regions[r]) for r in range(toy.EP)]), d["regions_digest"])


def test_native_apply_deliveries_error_paths():
    regions = np.zeros((2, 16), np.uint8)
    counters = np.zeros((2, 4), np.int64)
    msgs = dict(t_del=np.zeros(1, np.int64), src=np.zeros(1, np.int64), dst=np.ones(1, np.int64),
                src_off=np.zeros(1, np.int64), dst_off=np.zeros(1, np.int64), length=np.zeros(1, np.int64),
                op_hw=np.zeros(1, np.int64), imm=np.array([imm.encode_ll(0, 9, 0)], np.int64),
                work=np.zeros(1, np.int64))
    res, _, _ = _run_native_apply(regions, counters, 4, 0, 0, msgs, 2, 4, 2)
    assert res[2] == kernels.ERR_BAD_COUNTER and res[3] == 0
    msgs["length"] = np.array([64], np.int64)  # payload beyond the region
    msgs["imm"] = np.array([imm.encode_ll(0, 0, 0)], np.int64)
    res, _, _ = _run_native_apply(regions, counters, 4, 0, 0, msgs, 2, 4, 2)
    assert res[2] == kernels.ERR_FAULT
    # HT stale sequence
    msgs = dict(msgs, length=np.zeros(1, np.int64), imm=np.array([imm.encode_ht(0, 0, 40000)], np.int64))
    res, _, _ = _run_native_apply(regions, counters, 4, 0, 1, msgs, 2, 4, 2)
    assert res[2] == kernels.ERR_HT_STALE_SEQ


# --- FifoChannel semantics ---------------------------------------
def test_fifo_examples():
    ch = FifoChannel(2, spin=0)
    a = command.TransferCmd(command.WRITE, dst_rank=3, length_or_value=7168)
    b = command.TransferCmd(command.ATOMIC, dst_rank=1, length_or_value=5)
    assert ch.poll() is None
    assert ch.push(a) == 0 and ch.push(b) == 1
    with pytest.raises(ProtocolViolation):
        ch.push(a, block=False)  # capacity 2: the third push blocks
    assert ch.poll() == a and ch.poll() == a
    assert not ch.check_completion(0)
    assert ch.pop() == a and ch.pop() == b
    with pytest.raises(ProtocolViolation):
        ch.pop()
    ch.mark_completed(0)
    assert ch.check_completion(0) and not ch.check_completion(1)
    ch.mark_completed(1)
    ch.mark_completed(0)  # monotone
    assert ch.completed_upto == 1
    with pytest.raises(ProtocolViolation):
        ch.mark_completed(5)  # beyond head
    ch.shutdown()
    with pytest.raises(ChannelShutdown):
        ch.push(a)


def test_fifo_model_check_random_interleaving():
    g = np.random.default_rng(3)
    ch = FifoChannel(4, spin=0)
    oracle, pushed = [], 0
    for _ in range(10000):
        if g.random() < 0.5:
            c = command.TransferCmd(int(g.integers(0, 4)), int(g.integers(0, 4096)), int(g.integers(0, 64)),
                                    int(g.integers(0, 1 << 32)), int(g.integers(0, 1 << 32)),
                                    int(g.integers(0, 1 << 32)), int(g.integers(0, 4)))
            if len(oracle) < 4:
                assert ch.push(c, block=False) == pushed
                pushed += 1
                oracle.append(c)
            else:
                with pytest.raises(ProtocolViolation):
                    ch.push(c, block=False)
        else:
            if oracle:
                assert ch.poll() == oracle[0]
                assert ch.pop() == oracle.pop(0)
            else:
                assert ch.poll() is None
        assert 0 <= ch.tail - ch.head <= 4


def test_fifo_two_thread_stress_one_million():
    """SPEC.md:58 / :104 / :554: 1e6 commands through one ring (and 8 rings concurrently)
    with no loss, duplication or reordering; aggregate rate reported."""
    n, cap = 1_000_000, 64
    g = np.random.default_rng(0)
    lo = g.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)
    hi = g.integers(0, 1 << 54, n, dtype=np.int64)

    def run(ctl, lo_out, hi_out):
        def producer():
            done = 0
            while done < n:
                done += kernels.push_batch(ctl, cap, lo, hi, done, n - done, 1 << 16)

        def consumer():
            done = 0
            while done < n:
                done += kernels.pop_batch(ctl, cap, lo_out, hi_out, done, n - done, 1 << 16)
        ts = [threading.Thread(target=producer), threading.Thread(target=consumer)]
        for t in ts:
            t.start()
        return ts

    channels = 8
    ctls = [np.zeros(kernels.ctl_words(cap), np.int64) for _ in range(channels)]
    outs = [(np.zeros(n, np.int64), np.zeros(n, np.int64)) for _ in range(channels)]
    t0 = time.perf_counter()
    threads = [t for c, o in zip(ctls, outs) for t in run(c, *o)]
    for t in threads:
        t.join()
    dt = time.perf_counter() - t0
    for (lo_out, hi_out), ctl in zip(outs, ctls):
        assert np.array_equal(lo_out, lo) and np.array_equal(hi_out, hi)
        assert ctl[kernels.CTL_TAIL] == ctl[kernels.CTL_HEAD] == n
    rate = channels * n / dt
    print(f"FIFO stress: {channels} channels x {n} cmds, {rate / 1e6:.1f} Mcmd/s aggregate")
    assert rate > 1e6  # SPEC.md:554 smoke floor
