// deliveries.cpp — receiver-side delivery application, C++ port of the
// reference's ordering engine (kernels.py:124-318).
//
// Walks deliveries in the given (delivery-time) order and, per message:
//   1. lands the payload (regions[dst][dst_off..] <- regions[src][src_off..])
//      before any ordering check (kernels.py:164-167);
//   2. hardware atomic: counters[dst][dst_off/8] += length (kernels.py:168-180);
//   3. barrier imm kinds (>= 2) are escalated to the caller (kernels.py:183-186);
//   4. LL mode: per-(dst, src, counter) write counts; a fence atomic with
//      operand X is held until X writes arrived (kernels.py:187-248);
//   5. HT mode: per-(dst, src, channel) 16-bit sequence cursor with a pending
//      window; in-order messages apply and drain the window (kernels.py:249-318).
// Effects are appended to the eight caller-provided columns exactly as the
// reference does, so the effect trace compares element-for-element.
//
// Deliberate differences (documented in DESIGN.md): out-of-bounds payloads,
// counters and effect overflow return an error code instead of raising a
// numpy IndexError / writing out of bounds (reference quirk 4).
#include <cstdint>
#include <cstring>

#include "ctx.h"

namespace {

enum : int64_t { EFF_LL_WRITE = 0, EFF_LL_ATOMIC = 1, EFF_HT_DATA = 2, EFF_HT_ATOMIC = 3, EFF_HW_ATOMIC = 4 };
enum : int64_t {
  ERR_OK = 0,
  ERR_BAD_COUNTER = 1,
  ERR_LL_PENDING_OVERFLOW = 2,
  ERR_HT_STALE_SEQ = 3,
  ERR_HT_DUP_SLOT = 4,
  ERR_HT_WINDOW_OVERFLOW = 5,
  ERR_BAD_IMM_KIND = 6,
  ERR_FAULT = EPB_DLV_ERR_FAULT,
  ERR_EFFECT_OVERFLOW = EPB_DLV_ERR_EFFECT_OVERFLOW,
};
constexpr int64_t kSeqMod = 1 << 16;
constexpr int64_t kSeqWindow = 1 << 15;

struct EffectSink {
  int64_t *t, *kind, *dst, *src, *key, *aux, *counter, *work;
  int64_t cap, n = 0;
  bool push(int64_t vt, int64_t vk, int64_t vd, int64_t vs, int64_t vkey, int64_t vaux, int64_t vc, int64_t vw) {
    if (n >= cap) return false;
    t[n] = vt; kind[n] = vk; dst[n] = vd; src[n] = vs;
    key[n] = vkey; aux[n] = vaux; counter[n] = vc; work[n] = vw;
    ++n;
    return true;
  }
};

struct Engine {
  uint8_t* regions;
  int64_t ep, region_len;
  int64_t* counters;
  int64_t n_counters, n_counters_used, counter_base;
  const int64_t* imm_arr;
  const int64_t* work_id;
  int64_t* ll_counts;
  int32_t *ll_pend_x, *ll_pend_d, *ll_pend_n;
  int64_t pmax;
  int64_t* ht_applied;
  int32_t* ht_pend;
  int64_t nch, wmax;
  EffectSink eff;

  int64_t& counter(int64_t d, int64_t c) { return counters[d * n_counters + c]; }
  size_t llx(int64_t d, int64_t s, int64_t c) const { return ((size_t)d * ep + s) * n_counters + c; }
  size_t htx(int64_t d, int64_t s, int64_t c) const { return ((size_t)d * ep + s) * nch + c; }

  // kernels.py:285-318 — apply one in-order HT message (data or ring atomic).
  int64_t ht_apply(int64_t j, int64_t t_now, int64_t d, int64_t s) {
    const int64_t imm = imm_arr[j];
    const int64_t kind = imm & 3, ch = (imm >> 2) & 0x3F, seq = (imm >> 8) & 0xFFFF, operand = (imm >> 24) & 0xFF;
    if (kind == 0) {
      if (!eff.push(t_now, EFF_HT_DATA, d, s, ch, seq, 0, work_id[j])) return ERR_EFFECT_OVERFLOW;
    } else {
      const int64_t role_head = (operand & 0x80) ? 1 : 0;
      const int64_t cidx = counter_base + (s * nch + ch) * 2 + role_head;
      if (cidx < 0 || cidx >= n_counters) return ERR_BAD_COUNTER;
      counter(d, cidx) += operand & 0x7F;
      if (!eff.push(t_now, EFF_HT_ATOMIC, d, s, ch, seq, counter(d, cidx), work_id[j])) return ERR_EFFECT_OVERFLOW;
    }
    ht_applied[htx(d, s, ch)] += 1;
    return ERR_OK;
  }
};

}  // namespace

extern "C" int epb_apply_deliveries(uint8_t* regions, int64_t ep, int64_t region_len, int64_t* counters,
                                    int64_t n_counters, int64_t n_counters_used, int64_t counter_base,
                                    int64_t mode_ht, int64_t n, const int64_t* t_del, const int64_t* src_rank,
                                    const int64_t* dst_rank, const int64_t* src_off, const int64_t* dst_off,
                                    const int64_t* length, const int64_t* op_hw, const int64_t* imm_arr,
                                    const int64_t* work_id, int64_t* ll_counts, int32_t* ll_pend_x,
                                    int32_t* ll_pend_d, int32_t* ll_pend_n, int64_t pmax, int64_t* ht_applied,
                                    int32_t* ht_pend, int64_t n_channels, int64_t wmax, int64_t* eff_t,
                                    int64_t* eff_kind, int64_t* eff_dst, int64_t* eff_src, int64_t* eff_key,
                                    int64_t* eff_aux, int64_t* eff_counter, int64_t* eff_work, int64_t eff_cap,
                                    int64_t* esc_idx, int64_t esc_cap, int64_t* result4) {
  Engine E{regions, ep, region_len, counters, n_counters, n_counters_used, counter_base, imm_arr, work_id,
           ll_counts, ll_pend_x, ll_pend_d, ll_pend_n, pmax, ht_applied, ht_pend, n_channels, wmax,
           EffectSink{eff_t, eff_kind, eff_dst, eff_src, eff_key, eff_aux, eff_counter, eff_work, eff_cap}};
  int64_t nesc = 0;
  auto finish = [&](int64_t err, int64_t bad) {
    result4[0] = E.eff.n;
    result4[1] = nesc;
    result4[2] = err;
    result4[3] = bad;
    return EPB_OK;
  };

  for (int64_t i = 0; i < n; ++i) {
    const int64_t s = src_rank[i], d = dst_rank[i], ln = length[i];
    if (s < 0 || s >= ep || d < 0 || d >= ep) return finish(ERR_FAULT, i);
    if (ln > 0) {  // payload lands first (kernels.py:164-167)
      if (src_off[i] < 0 || dst_off[i] < 0 || src_off[i] + ln > region_len || dst_off[i] + ln > region_len)
        return finish(ERR_FAULT, i);
      std::memmove(regions + d * region_len + dst_off[i], regions + s * region_len + src_off[i], (size_t)ln);
    }
    if (op_hw[i] != 0) {  // hardware atomic: operand rides in length (kernels.py:168-180)
      const int64_t cidx = dst_off[i] / 8;
      if (cidx < 0 || cidx >= n_counters) return finish(ERR_BAD_COUNTER, i);
      E.counter(d, cidx) += ln;
      if (!E.eff.push(t_del[i], EFF_HW_ATOMIC, d, s, cidx, ln, E.counter(d, cidx), work_id[i]))
        return finish(ERR_EFFECT_OVERFLOW, i);
      continue;
    }
    const int64_t imm = imm_arr[i], kind = imm & 3;
    if (kind >= 2) {  // barrier words go to the protocol layer (kernels.py:183-186)
      if (nesc >= esc_cap) return finish(ERR_EFFECT_OVERFLOW, i);
      esc_idx[nesc++] = i;
      continue;
    }
    if (mode_ht == 0) {
      const int64_t cidx = (imm >> 2) & 0x3FF, operand = (imm >> 12) & 0xFFFFF;
      if (cidx >= n_counters_used || counter_base + cidx >= n_counters) return finish(ERR_BAD_COUNTER, i);
      const size_t k3 = E.llx(d, s, cidx);
      if (kind == 0 || ln > 0) {  // counted write (kernels.py:193-208)
        ll_counts[k3] += 1;
        if (!E.eff.push(t_del[i], EFF_LL_WRITE, d, s, cidx, ll_counts[k3], E.counter(d, counter_base + cidx),
                        work_id[i]))
          return finish(ERR_EFFECT_OVERFLOW, i);
        // release deferred fences whose X is now met (kernels.py:210-232): swap-remove scan
        int32_t* px = ll_pend_x + k3 * pmax;
        int32_t* pd = ll_pend_d + k3 * pmax;
        for (int32_t j = 0; j < ll_pend_n[k3];) {
          if (px[j] <= ll_counts[k3]) {
            E.counter(d, counter_base + cidx) += pd[j];
            if (!E.eff.push(t_del[i], EFF_LL_ATOMIC, d, s, cidx, px[j], E.counter(d, counter_base + cidx), -1))
              return finish(ERR_EFFECT_OVERFLOW, i);
            const int32_t last = ll_pend_n[k3] - 1;
            px[j] = px[last];
            pd[j] = pd[last];
            ll_pend_n[k3] = last;
          } else {
            ++j;
          }
        }
      }
      if (kind == 1) {  // fence atomic (kernels.py:233-248)
        const int64_t x = operand, delta = ln > 0 ? 1 : operand;
        if (ll_counts[k3] >= x) {
          E.counter(d, counter_base + cidx) += delta;
          if (!E.eff.push(t_del[i], EFF_LL_ATOMIC, d, s, cidx, x, E.counter(d, counter_base + cidx), work_id[i]))
            return finish(ERR_EFFECT_OVERFLOW, i);
        } else {
          const int32_t p = ll_pend_n[k3];
          if (p >= pmax) return finish(ERR_LL_PENDING_OVERFLOW, i);
          ll_pend_x[k3 * pmax + p] = (int32_t)x;
          ll_pend_d[k3 * pmax + p] = (int32_t)delta;
          ll_pend_n[k3] = p + 1;
        }
      }
    } else {
      const int64_t ch = (imm >> 2) & 0x3F, seq = (imm >> 8) & 0xFFFF;
      if (ch >= n_channels) return finish(ERR_BAD_COUNTER, i);
      const size_t k3 = E.htx(d, s, ch);
      const int64_t expected = ht_applied[k3] % kSeqMod;
      const int64_t dseq = ((seq - expected) % kSeqMod + kSeqMod) % kSeqMod;
      if (dseq >= kSeqWindow) return finish(ERR_HT_STALE_SEQ, i);
      if (dseq == 0) {
        if (int64_t e = E.ht_apply(i, t_del[i], d, s)) return finish(e, i);
        while (true) {  // drain consecutive deferred messages (kernels.py:262-274)
          const int64_t slot = ht_applied[k3] % wmax;
          const int32_t pend = ht_pend[k3 * wmax + slot];
          if (pend == 0) break;
          ht_pend[k3 * wmax + slot] = 0;
          if (int64_t e = E.ht_apply(pend - 1, t_del[i], d, s)) return finish(e, i);
        }
      } else {
        if (dseq >= wmax) return finish(ERR_HT_WINDOW_OVERFLOW, i);
        const int64_t slot = (ht_applied[k3] + dseq) % wmax;
        if (ht_pend[k3 * wmax + slot] != 0) return finish(ERR_HT_DUP_SLOT, i);
        ht_pend[k3 * wmax + slot] = (int32_t)(i + 1);
      }
    }
  }
  return finish(ERR_OK, -1);
}
