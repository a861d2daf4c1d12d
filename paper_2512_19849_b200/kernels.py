"""Host hot loops with the reference's exact signatures (drop-in for epsim.kernels).

* ``push_batch`` / ``pop_batch``  -> epb_ring_push_batch / epb_ring_pop_batch (ring.cpp),
  same control-array layout (kernels.py:23-31) and batch semantics
  (kernels.py:61-104), with release/acquire counters; GIL released during the call.
* ``apply_deliveries``            -> epb_apply_deliveries (deliveries.cpp), same 29
  positional arguments and (n_effects, n_escalated, err, bad_index) result
  (kernels.py:124-282).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib, nptr
from .errors import ChannelShutdown

CTL_TAIL, CTL_HEAD, CTL_COMPLETED, CTL_FLAGS, CTL_SLOT0 = 0, 8, 16, 24, 32
FLAG_SHUTDOWN = 1
EFF_LL_WRITE, EFF_LL_ATOMIC, EFF_HT_DATA, EFF_HT_ATOMIC, EFF_HW_ATOMIC = range(5)
(ERR_OK, ERR_BAD_COUNTER, ERR_LL_PENDING_OVERFLOW, ERR_HT_STALE_SEQ, ERR_HT_DUP_SLOT, ERR_HT_WINDOW_OVERFLOW,
 ERR_BAD_IMM_KIND, ERR_FAULT, ERR_EFFECT_OVERFLOW) = range(9)
BACKEND = "native"


def ctl_words(capacity: int) -> int:
    return CTL_SLOT0 + 2 * capacity


def _p64(a):
    if not (isinstance(a, np.ndarray) and a.dtype == np.int64 and a.flags.c_contiguous):
        raise TypeError("expected a C-contiguous int64 numpy array")
    return nptr(a, C.c_int64)


def push_batch(ctl, cap, lo, hi, start, want, max_spin) -> int:
    r = lib.epb_ring_push_batch(_p64(ctl), int(cap), _p64(lo), _p64(hi), int(start), int(want), int(max_spin))
    if r < 0:
        raise ChannelShutdown("push refused: channel shut down")
    return int(r)


def pop_batch(ctl, cap, lo_out, hi_out, start, want, max_spin) -> int:
    return int(lib.epb_ring_pop_batch(_p64(ctl), int(cap), _p64(lo_out), _p64(hi_out), int(start), int(want),
                                      int(max_spin)))


def apply_deliveries(regions, counters, n_counters_used, counter_base, mode_ht, t_del, src_rank, dst_rank, src_off,
                     dst_off, length, op_hw, imm_arr, work_id, ll_counts, ll_pend_x, ll_pend_d, ll_pend_n,
                     ht_applied, ht_pend, eff_t, eff_kind, eff_dst, eff_src, eff_key, eff_aux, eff_counter,
                     eff_work, esc_idx):
    ep, region_len = regions.shape
    n = t_del.shape[0]
    for a, dt in ((regions, np.uint8), (counters, np.int64), (ll_counts, np.int64), (ll_pend_x, np.int32),
                  (ll_pend_d, np.int32), (ll_pend_n, np.int32), (ht_applied, np.int64), (ht_pend, np.int32)):
        if a.dtype != dt or not a.flags.c_contiguous:
            raise TypeError("state arrays must be C-contiguous with the reference dtypes")
    msg = [np.ascontiguousarray(a, np.int64) for a in (t_del, src_rank, dst_rank, src_off, dst_off, length, op_hw,
                                                        imm_arr, work_id)]
    res = np.zeros(4, np.int64)
    check(lib.epb_apply_deliveries(
        regions.ctypes.data, ep, region_len, _p64(counters), counters.shape[1], int(n_counters_used),
        int(counter_base), int(mode_ht), n, *[_p64(a) for a in msg], _p64(ll_counts),
        nptr(ll_pend_x, C.c_int32), nptr(ll_pend_d, C.c_int32), nptr(ll_pend_n, C.c_int32), ll_pend_x.shape[3],
        _p64(ht_applied), nptr(ht_pend, C.c_int32), ht_applied.shape[2], ht_pend.shape[3],
        *[_p64(a) for a in (eff_t, eff_kind, eff_dst, eff_src, eff_key, eff_aux, eff_counter, eff_work)],
        eff_t.shape[0], _p64(esc_idx), esc_idx.shape[0], _p64(res)))
    return int(res[0]), int(res[1]), int(res[2]), int(res[3])
