// chunked.cu — bounded chunked ring channels for the normal (high-throughput)
// path: ht_transport = EPB_HT_RING.
//
// Reference semantics: RingChannel (chunk-granular ring,
// 32-token chunks, a producer-advanced tail and a consumer-advanced head,
// tail - head <= slots, a slot is rewritten only after its head has passed),
// dispatch_ht over those rings (chunks per (destination,
// channel), a tail atomic after each chunk, the receiver returns credit by
// advancing the head, imm.py:28-31 HT_ROLE_HEAD) and the per-channel ordering
// of PAPER.md:348-357.
//
// B200 mapping.  Every rank owns, for each source rank and each lane, one
// ring in its symmetric region; a lane is a (sender block, receiver block)
// pair and covers a contiguous range of the count exchange's channels, i.e.
// a contiguous token range at every source.  The sender stores a chunk's rows
// into the receiver's ring over NVLink, then st.release.sys's the new tail
// (one 4-byte word in the receiver's Meta); the receiver acquires the tail,
// copies (dispatch) or reduces (combine) the slots, then st.release.sys's the
// new head into the sender's Meta.  Tails and heads are cumulative u32 token
// counts (rings are a power of two long), so rings carry over across calls
// without a reset.  Per-ring order is the token order, so the receiver never
// reorders: the dispatch slot carries the row's final receive index, the
// combine receiver takes each contributing rank's next slot.
//
// The rings bound the arena to R x lanes x ring_tokens slots (the worst-case
// receive slots of the direct path hold R x T rows); the receive tensors are
// ordinary device memory sized from the notified counts.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "ctx.h"

namespace epb {

constexpr int kRingThreads = 512;  // 16 warps
constexpr int kRingChunk = 32;     // tokens per chunk
constexpr int kRingUnroll = 7;     // 16-byte words per lane in flight per row pass

struct RingGeom {
  int lanes, ring_tokens;
  int64_t disp_slot, comb_slot, disp_off, comb_off;
  // dispatch slot fields: row | scales | topk idx | topk weights | src idx | receive row | canary
  int64_t o_sc, o_ti, o_tw, o_src, o_row, o_can;
  int64_t comb_can;  // combine slot: row | weights | canary
  // test hook (EPB_RING_UNSAFE_NO_CREDIT=1): the sender skips the credit wait,
  // so it overruns unread slots and the canaries must catch it
  int no_credit;
};

struct RingDispatchParams {
  int n_local;
  RankView rv[kMaxLocal];
  epb_ring_dispatch_args_t a[kMaxLocal];
  RingGeom g;
};

struct RingCombineParams {
  int n_local;
  RankView rv[kMaxLocal];
  epb_ring_combine_args_t a[kMaxLocal];
  RingGeom g;
};

__device__ __forceinline__ char* ring_at(char* region, const RingGeom& g, int kind, int src, int lane) {
  const int64_t off = kind == 0 ? g.disp_off : g.comb_off;
  const int64_t slot = kind == 0 ? g.disp_slot : g.comb_slot;
  return region + off + ((int64_t)src * g.lanes + lane) * g.ring_tokens * slot;
}

// Channels [c_lo, c_hi) of the count exchange handled by lane l, and their tokens.
__device__ __forceinline__ void lane_range(int l, int lanes, int C, int T, int& c_lo, int& c_hi, int& t_lo,
                                           int& t_hi) {
  const int Tc = (T + C - 1) / C;
  c_lo = l * C / lanes;
  c_hi = (l + 1) * C / lanes;
  t_lo = min(T, c_lo * Tc);
  t_hi = min(T, c_hi * Tc);
}

// Rows from source s that fall in channels [c_lo, c_hi): [first, first + n) of s's run at me.
__device__ __forceinline__ void lane_rows(const int32_t* rcp, int C, int s, int c_lo, int c_hi, int& first, int& n) {
  first = c_lo > 0 ? rcp[s * C + c_lo - 1] : 0;
  n = c_hi > c_lo ? rcp[s * C + c_hi - 1] - first : 0;
}

__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Producer side: wait until the ring has room for n more slots.
__device__ __forceinline__ void wait_credit(const RankView& rv, const uint32_t* head, uint32_t sent, int n, int cap,
                                            int64_t tag) {
  uint64_t t0 = 0;
  int iter = 0;
  while ((int32_t)(sent + (uint32_t)n - ld_acquire_sys(head)) > cap) {
    if ((++iter & 1023) == 0) {
      const uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > rv.timeout_ns) {
        report_error(rv, EPB_ERR_DEADLOCK, tag);
        return;
      }
    }
  }
}

// Copy one row of n16 16-byte words (kNcSrc: the source is read-only input).
template <bool kNcSrc>
__device__ __forceinline__ void copy_row(const int4* src, int4* dst, int n16, int lane) {
  for (int base = 0; base < n16; base += 32 * kRingUnroll) {
    int4 v[kRingUnroll];
#pragma unroll
    for (int u = 0; u < kRingUnroll; ++u) {
      const int i = base + u * 32 + lane;
      if (i < n16) v[u] = kNcSrc ? ld_nc_v4(src + i) : ld_cg_v4(src + i);
    }
#pragma unroll
    for (int u = 0; u < kRingUnroll; ++u) {
      const int i = base + u * 32 + lane;
      if (i < n16) st_v4(dst + i, v[u]);
    }
  }
}

// ---------------------------------------------------------------------------
// dispatch: block 2l sends lane l's tokens to every destination (one warp
// group per destination), block 2l+1 drains lane l's ring of every source
// (one warp group per source) into the receive tensors.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRingThreads, 1) ring_dispatch_kernel(const __grid_constant__ RingDispatchParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_ring_dispatch_args_t& a = P.a[lr];
  const RingGeom& g = P.g;
  const int R = rv.world, me = rv.rank, l = blockIdx.x >> 1, role = blockIdx.x & 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int ng = min(R, nwarps), gw = nwarps / ng, grp = warp / gw, wig = warp % gw;
  if (grp >= ng) return;
  const int C = a.num_channels, T = a.num_tokens, RT = g.ring_tokens;
  int c_lo, c_hi, t_lo, t_hi;
  lane_range(l, g.lanes, C, T, c_lo, c_hi, t_lo, t_hi);
  Scratch* sc = scratch_of(rv.base);
  Meta* my = meta_of(rv.base);
  const int64_t row_bytes = (int64_t)a.hidden * a.elem_bytes;
  const int n16 = (int)(row_bytes >> 4), k = a.num_topk, S = a.num_scales;
  const int L = (a.topk_idx != nullptr && a.num_experts > 0) ? a.num_experts / R : 0;
  __shared__ uint32_t s_m[kMaxRanks];

  if (role == 0) {
    for (int d = grp; d < R; d += ng) {
      uint32_t sent = sc->rc_sent[0][d][l];
      uint32_t published = sent;  // tail value last released
      char* ring = ring_at(rv.peer[d], g, 0, me, l);
      uint32_t* tail = &meta_of(rv.peer[d])->rc_tail[0][me][l];
      const int base_d = me > 0 ? a.rank_prefix_matrix[(me - 1) * R + d] : 0;
      for (int w0 = t_lo; w0 < t_hi; w0 += kRingChunk) {
        const int t = w0 + lane;
        const int sh = t < t_hi ? a.send_head[(size_t)t * R + d] : -1;
        const unsigned b = __ballot_sync(0xffffffffu, sh >= 0);
        const int n = __popc(b);
        if (n == 0) continue;
        if (wig == 0 && lane == 0 && !g.no_credit) wait_credit(rv, &my->rc_head[0][d][l], sent, n, RT, 0x900 + d);
        group_sync(1 + grp, gw * 32);
        for (int j = wig; j < n; j += gw) {
          const int tj = __fns(b, 0, j + 1);
          const int tt = w0 + tj;
          const int shj = __shfl_sync(0xffffffffu, sh, tj);
          char* slot = ring + (int64_t)((sent + (uint32_t)j) & (uint32_t)(RT - 1)) * g.disp_slot;
          copy_row<true>(reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + (size_t)tt * row_bytes),
                         reinterpret_cast<int4*>(slot), n16, lane);
          if (a.x_scales != nullptr)
            for (int i = lane; i < S; i += 32)
              reinterpret_cast<float*>(slot + g.o_sc)[i] = a.x_scales[(size_t)tt * S + i];
          if (a.topk_idx != nullptr && lane < k) {
            const int64_t e = a.topk_idx[(size_t)tt * k + lane];
            const int64_t le = (e >= (int64_t)d * L && e < (int64_t)(d + 1) * L) ? e - (int64_t)d * L : -1;
            reinterpret_cast<int64_t*>(slot + g.o_ti)[lane] = le;
            reinterpret_cast<float*>(slot + g.o_tw)[lane] =
                (a.topk_weights != nullptr && le >= 0) ? a.topk_weights[(size_t)tt * k + lane] : 0.0f;
          }
          if (lane == 0) {
            *reinterpret_cast<int32_t*>(slot + g.o_src) = tt;
            *reinterpret_cast<int32_t*>(slot + g.o_row) = base_d + shj;
            // canary: the slot's cumulative sequence number in this ring (SPEC.md:470,
            // :477 "canary word per slot"); a slot overwritten before it was read
            // carries a sequence number RT (or more) ahead of what the receiver expects
            *reinterpret_cast<uint32_t*>(slot + g.o_can) = sent + (uint32_t)j;
          }
        }
        // the tail advances by whole 32-token chunks (32 tokens
        // -> one chunk write + one tail update, 33 -> two) and at the end; the
        // group's stores precede it (release cumulativity over the barrier)
        group_sync(1 + grp, gw * 32);
        sent += (uint32_t)n;
        if (wig == 0 && lane == 0 && (sent - published >= (uint32_t)kRingChunk || w0 + kRingChunk >= t_hi)) {
          st_release_sys(tail, sent);
          published = sent;
        }
      }
      if (wig == 0 && lane == 0 && published != sent) st_release_sys(tail, sent);
      if (wig == 0 && lane == 0) sc->rc_sent[0][d][l] = sent;
    }
  } else {
    for (int s = grp; s < R; s += ng) {
      int first, n_exp;
      lane_rows(a.recv_channel_prefix_matrix, C, s, c_lo, c_hi, first, n_exp);
      const uint32_t recvd = sc->rc_recvd[0][s][l];
      const char* ring = ring_at(rv.base, g, 0, s, l);
      uint32_t* head = &meta_of(rv.peer[s])->rc_head[0][me][l];
      int done = 0;
      if (g.no_credit && wig == 0 && lane == 0) {  // test hook: let the unthrottled sender lap the ring
        const uint64_t t_hold = globaltimer();
        while (globaltimer() - t_hold < 200000) __nanosleep(1000);
      }
      while (done < n_exp) {
        if (wig == 0 && lane == 0) {
          uint64_t t0 = 0;
          int iter = 0;
          int avail;
          while ((avail = (int)(ld_acquire_sys(&my->rc_tail[0][s][l]) - (recvd + (uint32_t)done))) <= 0) {
            if ((++iter & 1023) == 0) {
              const uint64_t now = globaltimer();
              if (t0 == 0) t0 = now;
              else if (now - t0 > rv.timeout_ns) {
                report_error(rv, EPB_ERR_DEADLOCK, 0x940 + s);
                avail = -1;  // give up on this ring: nothing it holds is trusted
                break;
              }
            }
          }
          s_m[grp] = avail < 0 ? 0xffffffffu : (uint32_t)min(avail, n_exp - done);
        }
        group_sync(1 + grp, gw * 32);
        if (s_m[grp] == 0xffffffffu) {  // timed out: skip the copy, release the credit, move on
          done = n_exp;
          if (wig == 0 && lane == 0) st_release_sys(head, recvd + (uint32_t)done);
          break;
        }
        const int m = (int)s_m[grp];
        for (int j = wig; j < m; j += gw) {
          const uint32_t seq = recvd + (uint32_t)(done + j);
          const char* slot = ring + (int64_t)(seq & (uint32_t)(RT - 1)) * g.disp_slot;
          int row = 0, bad = 0;
          if (lane == 0) {
            row = __ldcg(reinterpret_cast<const int32_t*>(slot + g.o_row));
            const uint32_t can = __ldcg(reinterpret_cast<const uint32_t*>(slot + g.o_can));
            if (can != seq) {  // an unread slot was overwritten (or never written)
              report_error(rv, EPB_ERR_INVARIANT, ((int64_t)0x9a0 << 40) | ((int64_t)s << 32) | can);
              bad = 1;
            } else if (row < 0 || row >= a.num_recv) {
              report_error(rv, EPB_ERR_FAULT, ((int64_t)0x9b0 << 40) | (uint32_t)row);
              bad = 1;
            }
          }
          if (__shfl_sync(0xffffffffu, bad, 0)) continue;
          row = __shfl_sync(0xffffffffu, row, 0);
          copy_row<false>(reinterpret_cast<const int4*>(slot),
                          reinterpret_cast<int4*>(static_cast<char*>(a.recv_x) + (size_t)row * row_bytes), n16, lane);
          if (a.recv_x_scales != nullptr)
            for (int i = lane; i < S; i += 32)
              a.recv_x_scales[(size_t)row * S + i] = __ldcg(reinterpret_cast<const float*>(slot + g.o_sc) + i);
          if (lane < k) {
            if (a.recv_topk_idx != nullptr)
              a.recv_topk_idx[(size_t)row * k + lane] = __ldcg(reinterpret_cast<const long long*>(slot + g.o_ti) + lane);
            if (a.recv_topk_weights != nullptr)
              a.recv_topk_weights[(size_t)row * k + lane] = __ldcg(reinterpret_cast<const float*>(slot + g.o_tw) + lane);
          }
          if (lane == 0) a.recv_src_idx[row] = __ldcg(reinterpret_cast<const int32_t*>(slot + g.o_src));
          // the row's stores consumed every lane's loads; the canary must still
          // hold this slot's sequence number (no overwrite while it was read)
          __syncwarp();
          if (lane == 0) {
            const uint32_t can = __ldcg(reinterpret_cast<const uint32_t*>(slot + g.o_can));
            if (can != seq) report_error(rv, EPB_ERR_INVARIANT, ((int64_t)0x9a1 << 40) | ((int64_t)s << 32) | can);
          }
        }
        // every read of these slots is done before the credit goes back
        group_sync(1 + grp, gw * 32);
        done += m;
        if (wig == 0 && lane == 0) st_release_sys(head, recvd + (uint32_t)done);
      }
      if (wig == 0 && lane == 0) sc->rc_recvd[0][s][l] = recvd + (uint32_t)n_exp;
    }
  }
}

// ---------------------------------------------------------------------------
// combine: block 2l returns, per source (warp group), the expert outputs of
// the rows that source's lane l sent me; block 2l+1 reduces lane l's tokens,
// taking each contributing rank's next slot (fp32, ascending rank order, one
// rounding to bf16 — the canonical order of SPEC.md:477).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRingThreads, 1) ring_combine_kernel(const __grid_constant__ RingCombineParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_ring_combine_args_t& a = P.a[lr];
  const RingGeom& g = P.g;
  const int R = rv.world, me = rv.rank, l = blockIdx.x >> 1, role = blockIdx.x & 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int C = a.num_channels, RT = g.ring_tokens, k = a.num_topk;
  const int64_t row_bytes = (int64_t)a.hidden * 2;
  const int n16 = (int)(row_bytes >> 4);
  Scratch* sc = scratch_of(rv.base);
  Meta* my = meta_of(rv.base);

  if (role == 0) {
    const int ng = min(R, nwarps), gw = nwarps / ng, grp = warp / gw, wig = warp % gw;
    if (grp >= ng) return;
    for (int s = grp; s < R; s += ng) {
      // rows source s sent me for its lane-l tokens: contiguous in my receive order
      int c_lo, c_hi, t_lo, t_hi;
      lane_range(l, g.lanes, C, 1 << 30, c_lo, c_hi, t_lo, t_hi);  // channel range only
      int first, n_rows;
      lane_rows(a.recv_channel_prefix_matrix, C, s, c_lo, c_hi, first, n_rows);
      const int j0 = (s > 0 ? a.rank_prefix_matrix[(s - 1) * R + me] : 0) + first;
      uint32_t sent = sc->rc_sent[1][s][l];
      char* ring = ring_at(rv.peer[s], g, 1, me, l);
      uint32_t* tail = &meta_of(rv.peer[s])->rc_tail[1][me][l];
      for (int w0 = 0; w0 < n_rows; w0 += kRingChunk) {
        const int n = min(kRingChunk, n_rows - w0);
        if (wig == 0 && lane == 0 && !g.no_credit) wait_credit(rv, &my->rc_head[1][s][l], sent, n, RT, 0x980 + s);
        group_sync(1 + grp, gw * 32);
        for (int j = wig; j < n; j += gw) {
          const int64_t row = j0 + w0 + j;
          char* slot = ring + (int64_t)((sent + (uint32_t)j) & (uint32_t)(RT - 1)) * g.comb_slot;
          copy_row<true>(reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + row * row_bytes),
                         reinterpret_cast<int4*>(slot), n16, lane);
          if (lane < k)
            reinterpret_cast<float*>(slot + row_bytes)[lane] =
                a.topk_weights != nullptr ? a.topk_weights[row * k + lane] : 0.0f;
          if (lane == 0) *reinterpret_cast<uint32_t*>(slot + g.comb_can) = sent + (uint32_t)j;  // canary
        }
        group_sync(1 + grp, gw * 32);
        sent += (uint32_t)n;
        if (wig == 0 && lane == 0) st_release_sys(tail, sent);
      }
      if (wig == 0 && lane == 0) sc->rc_sent[1][s][l] = sent;
    }
    return;
  }

  // receiver: my tokens of lane l, 32 at a time
  const int T = a.num_tokens;
  int c_lo, c_hi, t_lo, t_hi;
  lane_range(l, g.lanes, C, T, c_lo, c_hi, t_lo, t_hi);
  __shared__ uint32_t s_pos[kMaxRanks];   // slots of d's ring consumed so far (cumulative)
  __shared__ uint32_t s_bits[kMaxRanks];  // window tokens d contributes to
  if (tid < R) s_pos[tid] = sc->rc_recvd[1][tid][l];
  __syncthreads();
  for (int w0 = t_lo; w0 < t_hi; w0 += kRingChunk) {
    if (warp == 0) {
      const int t = w0 + lane;
      for (int d = 0; d < R; ++d) {
        const bool in = t < t_hi && a.send_head[(size_t)t * R + d] >= 0;
        const unsigned b = __ballot_sync(0xffffffffu, in);
        if (lane == 0) s_bits[d] = b;
      }
      __syncwarp();
      if (lane < R) {  // every contributing ring holds this window's slots
        const int d = lane, n = __popc(s_bits[d]);
        uint64_t t0 = 0;
        int iter = 0;
        while (n > 0 && (int32_t)(ld_acquire_sys(&my->rc_tail[1][d][l]) - (s_pos[d] + (uint32_t)n)) < 0) {
          if ((++iter & 1023) == 0) {
            const uint64_t now = globaltimer();
            if (t0 == 0) t0 = now;
            else if (now - t0 > rv.timeout_ns) {
              report_error(rv, EPB_ERR_DEADLOCK, 0x9c0 + d);
              break;
            }
          }
        }
      }
    }
    __syncthreads();
    for (int tt = warp; tt < kRingChunk && w0 + tt < t_hi; tt += nwarps) {
      const int t = w0 + tt;
      const char* src[kMaxRanks];
      int nv = 0;
      for (int d = 0; d < R; ++d) {
        const uint32_t b = s_bits[d];
        if (!((b >> tt) & 1u)) continue;
        const uint32_t idx = s_pos[d] + (uint32_t)__popc(b & ((1u << tt) - 1u));
        src[nv] = ring_at(rv.base, g, 1, d, l) + (int64_t)(idx & (uint32_t)(RT - 1)) * g.comb_slot;
        if (lane == 0) {
          const uint32_t can = __ldcg(reinterpret_cast<const uint32_t*>(src[nv] + g.comb_can));
          if (can != idx) report_error(rv, EPB_ERR_INVARIANT, ((int64_t)0x9c8 << 40) | ((int64_t)d << 32) | can);
        }
        ++nv;
      }
      int4* out = reinterpret_cast<int4*>(static_cast<char*>(a.combined_x) + (size_t)t * row_bytes);
      for (int i = lane; i < n16; i += 32) {
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
        for (int j = 0; j < nv; ++j) {
          const int4 v = ld_cg_v4(reinterpret_cast<const int4*>(src[j]) + i);
          const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[2 * q] = __fadd_rn(acc[2 * q], __uint_as_float(w[q] << 16));
            acc[2 * q + 1] = __fadd_rn(acc[2 * q + 1], __uint_as_float(w[q] & 0xffff0000u));
          }
        }
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
          o[q] = *reinterpret_cast<uint32_t*>(&h);
        }
        st_na_v4(out + i, make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]));
      }
      if (a.combined_topk_weights != nullptr && lane < k) {
        float wsum = 0.0f;
        for (int j = 0; j < nv; ++j) wsum = __fadd_rn(wsum, __ldcg(reinterpret_cast<const float*>(src[j] + row_bytes) + lane));
        a.combined_topk_weights[(size_t)t * k + lane] = wsum;
      }
    }
    __syncthreads();  // every read of the window's slots is done
    if (tid < R) {
      const int n = __popc(s_bits[tid]);
      if (n > 0) {
        s_pos[tid] += (uint32_t)n;
        st_release_sys(&meta_of(rv.peer[tid])->rc_head[1][me][l], s_pos[tid]);
      }
    }
    __syncthreads();
  }
  if (tid < R) sc->rc_recvd[1][tid][l] = s_pos[tid];
}

}  // namespace epb

using namespace epb;

static int ring_geometry(const epb_ctx* c, int hidden, int k, int lanes, int n_local, RingGeom* g,
                         epb_ring_layout_t* out) {
  if (hidden <= 0 || hidden % 128) return epb_set_error(EPB_ERR_CONFIG, "hidden must be a positive multiple of 128");
  if (k < 0 || k > 32) return epb_set_error(EPB_ERR_CONFIG, "num_topk must be in [0, 32]");
  if (lanes <= 0) lanes = std::max(1, std::min(kMaxLanes, c->num_sms / (2 * std::max(1, n_local))));
  if (lanes > kMaxLanes || 2 * lanes * n_local > c->num_sms)
    return epb_set_error(EPB_ERR_CONFIG, "ring lanes: 2 x lanes x local ranks must fit the SMs (<= 80 lanes)");
  const int64_t S = hidden / 128, R = c->world;
  std::memset(g, 0, sizeof(*g));
  g->lanes = lanes;
  g->o_sc = align_up(2 * (size_t)hidden, 16);
  g->o_ti = align_up(g->o_sc + S * 4, 8);
  g->o_tw = g->o_ti + 8 * k;
  g->o_src = g->o_tw + 4 * k;
  g->o_row = g->o_src + 4;
  g->o_can = g->o_row + 4;
  g->disp_slot = align_up(g->o_can + 4, 16);
  g->comb_can = 2 * (int64_t)hidden + 4 * (int64_t)k;
  g->comb_slot = align_up(g->comb_can + 4, 16);
  const char* nc = getenv("EPB_RING_UNSAFE_NO_CREDIT");
  g->no_credit = nc != nullptr && nc[0] == '1';
  const int64_t per_token = R * lanes * (g->disp_slot + g->comb_slot);
  int64_t rt = (int64_t)c->cfg.nvl_bytes / per_token;
  int pow2 = 0;
  while ((int64_t)1 << (pow2 + 1) <= rt && pow2 < 20) ++pow2;
  rt = (int64_t)1 << pow2;
  if (rt < 2 * kRingChunk)
    return epb_set_error(EPB_ERR_CONFIG, "ring transport: num_nvl_bytes too small for two 32-token chunks per ring");
  g->ring_tokens = (int)rt;
  g->disp_off = (int64_t)c->arena_off();
  g->comb_off = g->disp_off + R * lanes * rt * g->disp_slot;
  if (out) {
    out->lanes = lanes;
    out->ring_tokens = (int)rt;
    out->disp_slot_bytes = g->disp_slot;
    out->comb_slot_bytes = g->comb_slot;
    out->disp_off = g->disp_off;
    out->comb_off = g->comb_off;
    out->bytes_needed = rt * per_token;
  }
  return EPB_OK;
}

extern "C" int epb_ring_layout(epb_t* ctx, int hidden, int num_topk, int lanes, int n_local, epb_ring_layout_t* out) {
  if (!ctx || !out) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  RingGeom g;
  return ring_geometry(ctx, hidden, num_topk, lanes, n_local, &g, out);
}

static int ring_group_check(epb_t* const* ctxs, int n_local) {
  if (int e = check_group(ctxs, n_local)) return e;
  for (int i = 0; i < n_local; ++i)
    if (ctxs[i]->cfg.ht_transport != EPB_HT_RING)
      return epb_set_error(EPB_ERR_CONFIG, "ring calls need ht_transport = EPB_HT_RING on every rank");
  return EPB_OK;
}

extern "C" int epb_ring_dispatch(epb_t* const* ctxs, int n_local, const epb_ring_dispatch_args_t* args, int lanes,
                                 void* stream) {
  if (int e = ring_group_check(ctxs, n_local)) return e;
  RingDispatchParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_local = n_local;
  if (int e = ring_geometry(ctxs[0], args[0].hidden, args[0].num_topk, lanes, n_local, &P.g, nullptr)) return e;
  for (int i = 0; i < n_local; ++i) {
    const epb_ring_dispatch_args_t& a = args[i];
    if (a.elem_bytes != 1 && a.elem_bytes != 2) return epb_set_error(EPB_ERR_CONFIG, "elem_bytes must be 1 or 2");
    if (a.hidden != args[0].hidden || a.num_topk != args[0].num_topk)
      return epb_set_error(EPB_ERR_CONFIG, "all local ranks must share hidden and num_topk");
    if (a.num_channels <= 0 || a.num_channels > kMaxChannels) return epb_set_error(EPB_ERR_CONFIG, "bad num_channels");
    if (a.num_experts > 0 && a.num_experts % ctxs[i]->world)
      return epb_set_error(EPB_ERR_CONFIG, "num_experts must be a multiple of world");
    P.rv[i] = ctxs[i]->view();
    P.a[i] = a;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(epb_launch_grid_sync((void*)ring_dispatch_kernel, dim3(2 * P.g.lanes, n_local), dim3(kRingThreads), kargs,
                                0, st));
  return EPB_OK;
}

extern "C" int epb_ring_combine(epb_t* const* ctxs, int n_local, const epb_ring_combine_args_t* args, int lanes,
                                void* stream) {
  if (int e = ring_group_check(ctxs, n_local)) return e;
  RingCombineParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_local = n_local;
  if (int e = ring_geometry(ctxs[0], args[0].hidden, args[0].num_topk, lanes, n_local, &P.g, nullptr)) return e;
  for (int i = 0; i < n_local; ++i) {
    const epb_ring_combine_args_t& a = args[i];
    if (a.hidden != args[0].hidden || a.num_topk != args[0].num_topk)
      return epb_set_error(EPB_ERR_CONFIG, "all local ranks must share hidden and num_topk");
    if (a.num_channels <= 0 || a.num_channels > kMaxChannels) return epb_set_error(EPB_ERR_CONFIG, "bad num_channels");
    P.rv[i] = ctxs[i]->view();
    P.a[i] = a;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(epb_launch_grid_sync((void*)ring_combine_kernel, dim3(2 * P.g.lanes, n_local), dim3(kRingThreads), kargs,
                                0, st));
  return EPB_OK;
}

// Load this file's kernels now (see epb_preload_kernels, api.cpp).
cudaError_t epb_preload_chunked() {
  cudaFuncAttributes attr;
  for (const void* fn : {(const void*)ring_dispatch_kernel, (const void*)ring_combine_kernel})
    if (cudaError_t e = cudaFuncGetAttributes(&attr, fn)) return e;
  return cudaSuccess;
}
