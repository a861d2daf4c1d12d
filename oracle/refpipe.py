"""The reference's OWN CPU path, driven end to end — TEST/BENCH INFRASTRUCTURE ONLY.

``bench.py --impl reference`` times this module.  It runs the reference's
shipped code (``/root/reference/pkg/src/epsim``: ``command.pack_fields`` /
``unpack_fields``, ``imm.encode_ht_batch``, ``kernels.push_batch`` /
``pop_batch`` and ``kernels.apply_deliveries``), copied verbatim into
``oracle/_ref/epsim`` by ``build()`` (git-ignored; it travels to the GPU box
with the snapshot, where ``/root/reference`` does not exist).  Nothing here is
on the product path.

Pipeline per step (BASELINE.md "CPU baseline"):
  1. the HT dispatch delivery plan of SPEC.md:436-444 (one WRITE per (token,
     distinct destination rank), 32-token chunks per (src, dst, channel), a
     tail ATOMIC ``ht_atomic_operand(False, n)`` after each chunk; per-channel
     16-bit sequence numbers counting data and atomics) — built with numpy,
     not timed (the reference has no dispatch code that would produce it);
  2. ``command.pack_fields`` of every message                 (command.py:113-138)
  3. the SPSC ring, capacity 64, one producer and one consumer OS thread
     (``push_batch`` / ``pop_batch``, numba ``nogil``)         (kernels.py:61-104, :327-377)
  4. ``command.unpack_fields`` + ``imm.encode_ht_batch``         (command.py:141-158, imm.py:82-91)
  5. delivery-time sort with 50 % reordering
  6. ``kernels.apply_deliveries`` in HT mode: payload copy plus the per-channel
     in-order cursor                                          (kernels.py:124-318)
  7. combine: the reference has NO combine/reduce code (SPEC.md:446-454 is
     prose), so the canonical-order fp32 reduce of the numpy oracle port
     (oracle/ep.py combine) runs on the delivered rows.

Backend: numba via the cache shim of SURVEY.md Appendix A (numba cannot
``cache=True`` an ``exec``-generated function, kernels.py:386-409); the
reference files are not edited.
"""
from __future__ import annotations

import os
import shutil
import sys
import threading
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_OUT = HERE / "_ref"
REF_SRC = Path("/root/reference/pkg/src/epsim")
NCH = 8        # channels per (src, dst) pair (BASELINE.md CPU-baseline runs)
CHUNK = 32     # tokens per chunk
RING_CAP = 64  # SPSC capacity
WMAX = 1024    # HT reorder window per (src, dst, channel) cursor


def build_ref(src: Path = REF_SRC, out: Path = REF_OUT) -> bool:
    """Copy the reference's epsim package into oracle/_ref/epsim (the recipe
    ``__graft_entry__.build()`` runs; no source is edited).  Returns False when
    the reference is not present (the GPU box uses the copy shipped with the
    snapshot)."""
    if not src.is_dir():
        return False
    dst = out / "epsim"
    dst.mkdir(parents=True, exist_ok=True)
    for p in sorted(src.glob("*.py")):
        tgt = dst / p.name
        if not tgt.exists() or tgt.read_bytes() != p.read_bytes():
            shutil.copyfile(p, tgt)
    (out / "README").write_text("Verbatim copy of /root/reference/pkg/src/epsim made by oracle/refpipe.build_ref();\n"
                                "git-ignored build output, used only by bench.py --impl reference.\n")
    return True


_EPSIM = None


def load_epsim():
    """Import the copied reference with the numba cache shim; returns the module namespace."""
    global _EPSIM
    if _EPSIM is not None:
        return _EPSIM
    if not (REF_OUT / "epsim" / "kernels.py").exists():
        raise RuntimeError("oracle/_ref/epsim is missing: run __graft_entry__.build() where /root/reference exists")
    try:
        import numba
        if not getattr(numba.njit, "_epb_shim", False):
            orig = numba.njit

            def njit(*a, **kw):  # drop cache= for exec()-generated functions
                if a and callable(a[0]) and not kw:
                    return orig(*a)

                def deco(fn):
                    k = dict(kw)
                    if fn.__code__.co_filename == "<string>":
                        k.pop("cache", None)
                    return orig(**k)(fn)
                return deco
            njit._epb_shim = True
            numba.njit = njit
    except ImportError:
        os.environ["EPSIM_BACKEND"] = "numpy"
    if str(REF_OUT) not in sys.path:
        sys.path.insert(0, str(REF_OUT))
    from epsim import _backend, command, imm, kernels
    _EPSIM = type("epsim", (), dict(command=command, imm=imm, kernels=kernels, backend=_backend.BACKEND))
    return _EPSIM


def ht_plan(in_ranks, T: int, row: int, seed: int = 0):
    """HT dispatch delivery messages of every source (see module doc, step 1).

    in_ranks[s]: bool [T, R].  Region layout of SURVEY.md Appendix A:
    ``[send rows T*row][R*T*row receive area]``; source s's rows land at
    ``T*row + (s*T + pos)*row`` of the destination, pos = rank of the token
    among s's tokens for that destination.  Returns (columns, order by
    delivery time, t_del)."""
    R = len(in_ranks)
    per_ch = -(-T // NCH)
    cols = {k: [] for k in ("src", "dst", "kind", "ch", "seq", "operand", "src_off", "dst_off", "length")}
    for s in range(R):
        for d in range(R):
            toks = np.nonzero(in_ranks[s][:, d])[0]
            if not len(toks):
                continue
            pos = np.arange(len(toks))
            ch = toks // per_ch
            # position inside the (s, d, channel) stream, then chunk index
            first = np.searchsorted(ch, np.arange(NCH))
            p_in = pos - first[ch]
            chunk = p_in // CHUNK
            seq = p_in + chunk  # every earlier chunk of the channel added one tail atomic
            n = len(toks)
            cols["src"].append(np.full(n, s)); cols["dst"].append(np.full(n, d))
            cols["kind"].append(np.zeros(n, np.int64)); cols["ch"].append(ch); cols["seq"].append(seq)
            cols["operand"].append(np.zeros(n, np.int64))
            cols["src_off"].append(toks * row); cols["dst_off"].append(T * row + (s * T + pos) * row)
            cols["length"].append(np.full(n, row))
            # tail atomics: after each chunk, operand = tokens in that chunk
            cnt = np.bincount(ch, minlength=NCH)
            for c in range(NCH):
                nc = int(cnt[c])
                if nc == 0:
                    continue
                k = -(-nc // CHUNK)
                sizes = np.minimum(CHUNK, nc - np.arange(k) * CHUNK)
                a_seq = np.arange(k) * (CHUNK + 1) + sizes  # after the chunk's data messages
                cols["src"].append(np.full(k, s)); cols["dst"].append(np.full(k, d))
                cols["kind"].append(np.ones(k, np.int64)); cols["ch"].append(np.full(k, c)); cols["seq"].append(a_seq)
                cols["operand"].append(sizes)  # ht_atomic_operand(False, n) == n (imm.py:69-72)
                cols["src_off"].append(np.zeros(k, np.int64)); cols["dst_off"].append(np.zeros(k, np.int64))
                cols["length"].append(np.zeros(k, np.int64))
    out = {k: np.concatenate(v).astype(np.int64) for k, v in cols.items()}
    # posting order: per (src, dst, channel) stream by sequence number
    post = np.lexsort((out["seq"], out["ch"], out["dst"], out["src"]))
    out = {k: v[post] for k, v in out.items()}
    n = len(out["src"])
    g = np.random.default_rng(seed)
    t_post = np.arange(n, dtype=np.int64) * 10
    t_del = t_post + np.where(g.random(n) < 0.5, g.integers(1, 60, n) * 10 + 5, 0)
    order = np.lexsort((np.arange(n), t_del))
    return out, order, t_del


def _ring_transfer(k, lo, hi):
    """Move every command through one bounded SPSC ring: producer + consumer OS threads."""
    n = len(lo)
    ctl = np.zeros(k.ctl_words(RING_CAP), np.int64)
    lo_i, hi_i = lo.view(np.int64), hi.view(np.int64)
    lo_o, hi_o = np.zeros(n, np.int64), np.zeros(n, np.int64)

    def produce():
        done = 0
        while done < n:
            done += k.push_batch(ctl, RING_CAP, lo_i, hi_i, done, n - done, 1 << 20)

    th = threading.Thread(target=produce)
    th.start()
    got = 0
    while got < n:
        got += k.pop_batch(ctl, RING_CAP, lo_o, hi_o, got, n - got, 1 << 20)
    th.join()
    return lo_o.view(np.uint64), hi_o.view(np.uint64)


class HTDispatchStep:
    """One rank group's dispatch delivery through the reference + the oracle combine."""

    def __init__(self, xs, in_ranks, seed: int = 0):
        self.ep = load_epsim()
        self.R, (self.T, H) = len(xs), xs[0].shape
        self.row = 2 * H
        self.xs = xs
        self.in_ranks = in_ranks
        self.msgs, self.order, self.t_del = ht_plan(in_ranks, self.T, self.row, seed)
        self.region_len = self.T * self.row + self.R * self.T * self.row
        self.regions = np.zeros((self.R, self.region_len), np.uint8)
        for s in range(self.R):
            self.regions[s, : self.T * self.row] = xs[s].view(np.uint8).reshape(-1)
        self.n_ctr = 2 * self.R * NCH
        self.rows = int(sum(ir.sum() for ir in in_ranks))
        from concurrent.futures import ThreadPoolExecutor
        self.threads = max(1, len(os.sched_getaffinity(0)))
        self.pool = ThreadPoolExecutor(self.threads)
        self.tok_chunk = max(1, -(-self.T // self.threads))

    def run(self):
        """One timed step: returns the combined outputs (per source) after checking the delivery."""
        e, m = self.ep, self.msgs
        command, imm, kernels = e.command, e.imm, e.kernels
        n = len(m["src"])
        lo, hi = command.pack_fields(m["kind"], m["dst"], m["ch"], m["src_off"], m["dst_off"],
                                     np.where(m["kind"] == 1, m["operand"], m["length"]), np.zeros(n, np.int64))
        lo, hi = _ring_transfer(kernels, lo, hi)
        f = command.unpack_fields(lo, hi)
        imm_w = imm.encode_ht_batch(f["kind"], f["channel_id"], m["seq"], np.where(f["kind"] == 1, f["length_or_value"], 0))
        o = self.order
        length = np.where(f["kind"] == 1, 0, f["length_or_value"])
        counters = np.zeros((self.R, self.n_ctr), np.int64)
        ll_counts = np.zeros((self.R, self.R, 1), np.int64)
        ll_px = np.zeros((self.R, self.R, 1, 1), np.int32)
        ll_pd = np.zeros((self.R, self.R, 1, 1), np.int32)
        ll_pn = np.zeros((self.R, self.R, 1), np.int32)
        ht_applied = np.zeros((self.R, self.R, NCH), np.int64)
        ht_pend = np.zeros((self.R, self.R, NCH, WMAX), np.int32)
        cap = 2 * n + 16
        eff = [np.zeros(cap, np.int64) for _ in range(8)]
        esc = np.zeros(n, np.int64)
        res = kernels.apply_deliveries(
            self.regions, counters, self.n_ctr, 0, 1, self.t_del[o], m["src"][o], f["dst_rank"][o],
            f["src_offset"][o], f["dst_offset"][o], length[o], np.zeros(n, np.int64), imm_w[o],
            np.arange(n, dtype=np.int64)[o], ll_counts, ll_px, ll_pd, ll_pn, ht_applied, ht_pend, *eff, esc)
        if res[2] != 0:
            raise RuntimeError(f"reference apply_deliveries reported error {res}")
        return self._combine()

    def _recv(self, d):
        parts = []
        for s in range(self.R):
            nd = int(self.in_ranks[s][:, d].sum())
            off = self.T * self.row + s * self.T * self.row
            parts.append(self.regions[d, off: off + nd * self.row].view(np.uint16).reshape(nd, -1))
        return np.concatenate(parts, axis=0)

    def _combine(self):
        """The oracle port's canonical combine, token ranges spread over every host
        core (numpy releases the GIL in the gathers and adds)."""
        from oracle import ep as O
        recv = [self._recv(d) for d in range(self.R)]
        heads = []
        for s in range(self.R):
            ir = self.in_ranks[s]
            heads.append(np.where(ir, np.cumsum(ir, axis=0) - 1, -1).astype(np.int32))
        counts = np.array([[int(self.in_ranks[s][:, d].sum()) for d in range(self.R)] for s in range(self.R)])
        rpm = np.cumsum(counts, axis=0).astype(np.int32)
        jobs = [(s, a, min(a + self.tok_chunk, self.T)) for s in range(self.R) for a in range(0, self.T, self.tok_chunk)]
        parts = list(self.pool.map(
            lambda j: O.combine_rank(j[0], recv, self.in_ranks[j[0]][j[1]:j[2]], heads[j[0]][j[1]:j[2]], rpm)[0], jobs))
        out, i = [], 0
        for s in range(self.R):
            n = -(-self.T // self.tok_chunk)
            out.append(np.concatenate(parts[i:i + n], axis=0))
            i += n
        return recv, out


def time_steps(xs, in_ranks, steps: int, warmup: int, seed: int = 0):
    """(seconds per step, payload bytes per step [dispatch + combine rows], backend, host threads)."""
    st = HTDispatchStep(xs, in_ranks, seed)
    for _ in range(max(1, warmup)):
        st.run()
    t0 = time.perf_counter()
    for _ in range(steps):
        st.run()
    dt = (time.perf_counter() - t0) / max(1, steps)
    st.pool.shutdown()
    return dt, 2 * st.rows * st.row, st.ep.backend, st.threads
