"""Generate the golden fixtures by RUNNING THE REFERENCE (/root/reference/pkg/src/epsim).

Run in the development container (the reference does not exist on the GPU
box; the fixtures it writes are committed):

    EPSIM_BACKEND=numpy python tests/golden/make_golden.py

Fixtures (tests/golden/*.npz):
  codec.npz          command.pack_fields / unpack_fields / to_bytes + imm batch encoders
  ring.npz           a deterministic push/pop script on kernels.push_batch / pop_batch
  deliveries_kat.npz SPEC.md:345-347 examples through kernels.apply_deliveries
  ht_dispatch.npz    toy-config HT dispatch delivery through kernels.apply_deliveries
  ll_dispatch.npz    toy-config LL dispatch delivery through kernels.apply_deliveries
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("EPSIM_BACKEND", "numpy")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from epsim import command, errors, imm, kernels  # noqa: E402  (the reference)
from tests.golden import toy  # noqa: E402


def gen_codec():
    g = np.random.default_rng(1234)
    n = 4096
    f = dict(kind=g.integers(0, 4, n), dst_rank=g.integers(0, 4096, n), channel_id=g.integers(0, 64, n),
             src_offset=g.integers(0, 1 << 32, n, dtype=np.int64), dst_offset=g.integers(0, 1 << 32, n, dtype=np.int64),
             length_or_value=g.integers(0, 1 << 32, n, dtype=np.int64), flags=g.integers(0, 4, n))
    lo, hi = command.pack_fields(**f)
    back = command.unpack_fields(lo, hi)
    # scalar path + 16-byte records for the first 64
    recs = np.zeros((64, 16), np.uint8)
    for i in range(64):
        c = command.TransferCmd(**{k: int(v[i]) for k, v in f.items()})
        recs[i] = np.frombuffer(command.to_bytes(c), np.uint8)
        assert command.pack(c) == (int(lo[i]), int(hi[i]))
    kat = command.TransferCmd(kind=0, dst_rank=3, channel_id=5, src_offset=0x12345678, dst_offset=0xABCDEF01,
                              length_or_value=7168, flags=1)
    kat_lo, kat_hi = command.pack(kat)
    # reserved-bit rejection
    bad_hi = np.array([1 << 54, 1 << 63, (1 << 54) | 5], np.uint64)
    rejected = []
    for h in bad_hi:
        try:
            command.unpack(0, int(h))
            rejected.append(0)
        except errors.ProtocolViolation:
            rejected.append(1)
    # imm
    m = 2048
    ll_k, ll_c, ll_o = g.integers(0, 4, m), g.integers(0, 1024, m), g.integers(0, 1 << 20, m)
    ht_k, ht_c, ht_s, ht_o = g.integers(0, 4, m), g.integers(0, 64, m), g.integers(0, 1 << 20, m), g.integers(0, 256, m)
    np.savez_compressed(
        HERE / "codec.npz", **{f"f_{k}": np.asarray(v, np.int64) for k, v in f.items()},
        lo=lo, hi=hi, **{f"u_{k}": v for k, v in back.items()}, records=recs,
        kat=np.array([kat_lo, kat_hi], np.uint64), kat_bytes=np.frombuffer(command.to_bytes(kat), np.uint8),
        bad_hi=bad_hi, rejected=np.array(rejected),
        ll_k=ll_k, ll_c=ll_c, ll_o=ll_o, ll_out=imm.encode_ll_batch(ll_k, ll_c, ll_o),
        ht_k=ht_k, ht_c=ht_c, ht_s=ht_s, ht_o=ht_o, ht_out=imm.encode_ht_batch(ht_k, ht_c, ht_s, ht_o),
        imm_kat=np.array([imm.encode_ll(imm.ATOMIC, 7, 3), imm.encode_ht(imm.DATA, 3, 70000, 0x81),
                          *imm.decode_ht(imm.encode_ht(imm.DATA, 3, 70000, 0x81)), imm.seq_delta(1, 65535),
                          imm.ht_atomic_operand(True, 5)], np.int64))


def gen_ring():
    cap = 8
    ctl = np.zeros(kernels.ctl_words(cap), np.int64)
    g = np.random.default_rng(99)
    N = 200
    lo_src = g.integers(-(1 << 62), 1 << 62, N, dtype=np.int64)
    hi_src = g.integers(0, 1 << 54, N, dtype=np.int64)
    lo_out = np.zeros(N, np.int64)
    hi_out = np.zeros(N, np.int64)
    pushed = popped = 0
    script, results, snaps = [], [], []
    for step in range(120):
        if g.random() < 0.5:
            want = int(g.integers(0, 12))
            want = min(want, N - pushed)
            r = kernels.push_batch(ctl, cap, lo_src, hi_src, pushed, want, 0)
            pushed += r
            script.append((0, want))
        else:
            want = int(g.integers(0, 12))
            want = min(want, N - popped)
            r = kernels.pop_batch(ctl, cap, lo_out, hi_out, popped, want, 0)
            popped += r
            script.append((1, want))
        results.append(r)
        snaps.append(ctl.copy())
    np.savez_compressed(HERE / "ring.npz", cap=cap, lo_src=lo_src, hi_src=hi_src, script=np.array(script),
                        results=np.array(results), snaps=np.array(snaps), lo_out=lo_out, hi_out=hi_out)


def _run_apply(regions, counters, n_used, base, mode_ht, msgs, ep, nctr, nch, pmax=8, wmax=64):
    n = len(msgs["t_del"])
    ll_counts = np.zeros((ep, ep, nctr), np.int64)
    ll_px = np.zeros((ep, ep, nctr, pmax), np.int32)
    ll_pd = np.zeros((ep, ep, nctr, pmax), np.int32)
    ll_pn = np.zeros((ep, ep, nctr), np.int32)
    ht_applied = np.zeros((ep, ep, nch), np.int64)
    ht_pend = np.zeros((ep, ep, nch, wmax), np.int32)
    cap = 2 * n + 16
    eff = [np.zeros(cap, np.int64) for _ in range(8)]
    esc = np.zeros(n, np.int64)
    res = kernels.apply_deliveries(regions, counters, n_used, base, mode_ht, msgs["t_del"], msgs["src"],
                                   msgs["dst"], msgs["src_off"], msgs["dst_off"], msgs["length"], msgs["op_hw"],
                                   msgs["imm"], msgs["work"], ll_counts, ll_px, ll_pd, ll_pn, ht_applied, ht_pend,
                                   *eff, esc)
    ne = res[0]
    return res, np.stack([e[:ne] for e in eff]), esc[: res[1]], ll_counts, ht_applied


def gen_kat():
    """SPEC.md:345-347 examples."""
    out = {}
    # LL fence, X=3: w1, w2, A(X=3) deferred, w3 releases it; expert 7 independent of expert 3
    regions = np.zeros((2, 64), np.uint8)
    regions[0, :8] = np.arange(8)
    counters = np.zeros((2, 16), np.int64)
    msgs = dict(t_del=np.arange(6), src=np.zeros(6, np.int64), dst=np.ones(6, np.int64),
                src_off=np.array([0, 1, 0, 2, 0, 3]), dst_off=np.array([0, 1, 0, 2, 0, 3]),
                length=np.array([1, 1, 0, 1, 0, 1]), op_hw=np.zeros(6, np.int64),
                imm=np.array([imm.encode_ll(0, 3, 0), imm.encode_ll(0, 3, 0), imm.encode_ll(1, 3, 3),
                              imm.encode_ll(0, 3, 0), imm.encode_ll(1, 7, 0), imm.encode_ll(0, 7, 0)], np.int64),
                work=np.arange(6))
    res, eff, esc, llc, hta = _run_apply(regions, counters, 8, 0, 0, msgs, 2, 16, 4)
    out.update(ll_msgs=np.stack([msgs[k] for k in ("t_del", "src", "dst", "src_off", "dst_off", "length", "op_hw",
                                                   "imm", "work")]),
               ll_res=np.array(res), ll_eff=eff, ll_counters=counters, ll_regions=regions)
    # HT: arrivals seq 0, 1, 3(write), 2(write), 4(atomic)
    regions = np.zeros((2, 64), np.uint8)
    regions[0, :8] = np.arange(10, 18)
    counters = np.zeros((2, 32), np.int64)
    seqs = [0, 1, 3, 2, 4]
    kinds = [0, 0, 0, 0, 1]
    msgs = dict(t_del=np.arange(5), src=np.zeros(5, np.int64), dst=np.ones(5, np.int64),
                src_off=np.array([0, 1, 3, 2, 0]), dst_off=np.array([0, 1, 3, 2, 0]),
                length=np.array([1, 1, 1, 1, 0]), op_hw=np.zeros(5, np.int64),
                imm=np.array([imm.encode_ht(k, 2, s, imm.ht_atomic_operand(False, 5) if k else 0)
                              for k, s in zip(kinds, seqs)], np.int64), work=np.arange(5))
    res, eff, esc, llc, hta = _run_apply(regions, counters, 8, 0, 1, msgs, 2, 32, 4)
    out.update(ht_msgs=np.stack([msgs[k] for k in ("t_del", "src", "dst", "src_off", "dst_off", "length", "op_hw",
                                                   "imm", "work")]),
               ht_res=np.array(res), ht_eff=eff, ht_counters=counters, ht_regions=regions)
    np.savez_compressed(HERE / "deliveries_kat.npz", **out)


def gen_toy_dispatch():
    xs, idxs, ws = toy.make_inputs(0)
    L = toy.E // toy.EP
    # HT
    msgs, _ = toy.ht_plan(xs, idxs)
    regions = toy.regions_init(xs, toy.EP * toy.T)
    nctr = 2 * toy.EP * toy.NCH
    counters = np.zeros((toy.EP, nctr), np.int64)
    res, eff, esc, llc, hta = _run_apply(regions, counters, nctr, 0, 1, msgs, toy.EP, nctr, toy.NCH, wmax=512)
    assert res[2] == 0, res
    np.savez_compressed(HERE / "ht_dispatch.npz", msgs_digest=toy.msgs_digest(msgs), res=np.array(res), eff=eff,
                        counters=counters, ht_applied=hta, blocks=toy.ht_recv_blocks(regions, idxs),
                        regions_digest=np.stack([toy.digest_rows(regions[r]) for r in range(toy.EP)]))
    # LL
    msgs, _ = toy.ll_plan(xs, idxs)
    regions = toy.regions_init(xs, L * toy.EP * toy.T)
    counters = np.zeros((toy.EP, L), np.int64)
    res, eff, esc, llc, hta = _run_apply(regions, counters, L, 0, 0, msgs, toy.EP, L, toy.NCH, pmax=8)
    assert res[2] == 0, res
    np.savez_compressed(HERE / "ll_dispatch.npz", msgs_digest=toy.msgs_digest(msgs), res=np.array(res), eff=eff,
                        counters=counters, ll_counts=llc, blocks=toy.ll_recv_blocks(regions, idxs),
                        regions_digest=np.stack([toy.digest_rows(regions[r]) for r in range(toy.EP)]))


if __name__ == "__main__":
    from epsim import _backend
    print("reference backend:", _backend.BACKEND)
    gen_codec()
    gen_ring()
    gen_kat()
    gen_toy_dispatch()
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)
