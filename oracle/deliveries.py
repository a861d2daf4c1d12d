"""Oracle restatement of the receiver-side delivery application.

Semantics of kernels.py:124-318:
* payload lands before any ordering decision (kernels.py:164-167);
* hardware atomic adds `length` at counter dst_off//8 (kernels.py:168-180);
* imm kinds >= 2 escalate (kernels.py:183-186);
* LL: per (dst, src, counter) write counts; fence atomics wait for X writes;
  a write releases every deferred fence it satisfies, scanning with
  swap-with-last removal (kernels.py:187-248);
* HT: per (dst, src, channel) 16-bit cursor, pending window keyed by
  (cursor + delta) % WMAX, in-order message applies and drains (kernels.py:249-318).
Effects are returned as a list of 8-tuples (t, kind, dst, src, key, aux,
counter, work) in application order.  Pure Python: small cases only.
"""
from __future__ import annotations

import numpy as np

EFF_LL_WRITE, EFF_LL_ATOMIC, EFF_HT_DATA, EFF_HT_ATOMIC, EFF_HW_ATOMIC = range(5)
ERR_OK, ERR_BAD_COUNTER, ERR_LL_PENDING_OVERFLOW, ERR_HT_STALE_SEQ, ERR_HT_DUP_SLOT, ERR_HT_WINDOW_OVERFLOW = range(6)
SEQ_MOD, SEQ_WINDOW = 1 << 16, 1 << 15


class DeliveryState:
    def __init__(self, ep, n_counters, n_channels, pmax, wmax):
        self.ll_counts = np.zeros((ep, ep, n_counters), np.int64)
        self.ll_pending = {}  # (dst, src, cidx) -> list of [x, delta]
        self.pmax = pmax
        self.ht_applied = np.zeros((ep, ep, n_channels), np.int64)
        self.ht_window = {}  # (dst, src, ch) -> {slot: message index}
        self.wmax = wmax
        self.n_channels = n_channels


def apply(regions, counters, n_counters_used, counter_base, mode_ht, msgs, state: DeliveryState):
    """msgs: dict of equal-length int arrays t_del, src, dst, src_off, dst_off, length, op_hw, imm, work.
    Returns (effects, escalated, err, bad_index)."""
    eff, esc = [], []
    t_del, src_a, dst_a = msgs["t_del"], msgs["src"], msgs["dst"]
    so_a, do_a, ln_a, hw_a, imm_a, wk_a = (msgs[k] for k in ("src_off", "dst_off", "length", "op_hw", "imm", "work"))

    def ht_one(j, t_now, d, s):
        imm = int(imm_a[j])
        kind, ch, seq, opnd = imm & 3, (imm >> 2) & 63, (imm >> 8) & 0xFFFF, (imm >> 24) & 0xFF
        if kind == 0:
            eff.append((t_now, EFF_HT_DATA, d, s, ch, seq, 0, int(wk_a[j])))
        else:
            c = counter_base + 2 * (s * state.n_channels + ch) + (1 if opnd & 0x80 else 0)
            counters[d, c] += opnd & 0x7F
            eff.append((t_now, EFF_HT_ATOMIC, d, s, ch, seq, int(counters[d, c]), int(wk_a[j])))
        state.ht_applied[d, s, ch] += 1

    for i in range(len(t_del)):
        s, d, ln, t = int(src_a[i]), int(dst_a[i]), int(ln_a[i]), int(t_del[i])
        if ln > 0:
            o_s, o_d = int(so_a[i]), int(do_a[i])
            regions[d, o_d:o_d + ln] = regions[s, o_s:o_s + ln].copy()
        if hw_a[i]:
            c = int(do_a[i]) // 8
            counters[d, c] += ln
            eff.append((t, EFF_HW_ATOMIC, d, s, c, ln, int(counters[d, c]), int(wk_a[i])))
            continue
        imm = int(imm_a[i])
        kind = imm & 3
        if kind >= 2:
            esc.append(i)
            continue
        if not mode_ht:
            cidx, operand = (imm >> 2) & 0x3FF, imm >> 12
            if cidx >= n_counters_used:
                return eff, esc, ERR_BAD_COUNTER, i
            key = (d, s, cidx)
            pend = state.ll_pending.setdefault(key, [])
            if kind == 0 or ln > 0:
                state.ll_counts[key] += 1
                have = int(state.ll_counts[key])
                eff.append((t, EFF_LL_WRITE, d, s, cidx, have, int(counters[d, counter_base + cidx]), int(wk_a[i])))
                j = 0
                while j < len(pend):
                    if pend[j][0] <= have:
                        counters[d, counter_base + cidx] += pend[j][1]
                        eff.append((t, EFF_LL_ATOMIC, d, s, cidx, pend[j][0], int(counters[d, counter_base + cidx]), -1))
                        pend[j] = pend[-1]
                        pend.pop()
                    else:
                        j += 1
            if kind == 1:
                x = operand
                delta = 1 if ln > 0 else operand
                if state.ll_counts[key] >= x:
                    counters[d, counter_base + cidx] += delta
                    eff.append((t, EFF_LL_ATOMIC, d, s, cidx, x, int(counters[d, counter_base + cidx]), int(wk_a[i])))
                else:
                    if len(pend) >= state.pmax:
                        return eff, esc, ERR_LL_PENDING_OVERFLOW, i
                    pend.append([x, delta])
        else:
            ch, seq = (imm >> 2) & 63, (imm >> 8) & 0xFFFF
            cur = int(state.ht_applied[d, s, ch])
            delta = (seq - cur % SEQ_MOD) % SEQ_MOD
            if delta >= SEQ_WINDOW:
                return eff, esc, ERR_HT_STALE_SEQ, i
            win = state.ht_window.setdefault((d, s, ch), {})
            if delta == 0:
                ht_one(i, t, d, s)
                while True:
                    slot = int(state.ht_applied[d, s, ch]) % state.wmax
                    if slot not in win:
                        break
                    ht_one(win.pop(slot), t, d, s)
            else:
                if delta >= state.wmax:
                    return eff, esc, ERR_HT_WINDOW_OVERFLOW, i
                slot = (cur + delta) % state.wmax
                if slot in win:
                    return eff, esc, ERR_HT_DUP_SLOT, i
                win[slot] = i
    return eff, esc, ERR_OK, -1
