// normal.cu — high-throughput (normal-mode) EP path on sm_100a:
//   layout   : topk_idx -> per-rank / per-expert counts + is_token_in_rank
//   notify   : count all-gather over NVLink mailboxes + prefix sums
//   dispatch : dedup'd rows pushed straight into peers' receive slots
//   combine  : rows pushed back to their source, fp32 reduce in canonical
//              (ascending rank) order, bf16 out
//
// Semantics follow the reference's ep_engine spec: dedup per destination
// (SPEC.md:416-424), per-source token-ordered delivery
// (golden vectors from kernels.py:124-282 in
// tests/golden), canonical-order reduce.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "ctx.h"

namespace epb {

constexpr int kLayoutThreads = 256;
constexpr int kNotifyThreads = 1024;
constexpr int kDispatchThreads = 512;
constexpr int kCombineThreads = 512;
constexpr int kCopyUnroll = 7;  // 7 x 16 B per lane in flight = 3.5 KB per warp

// ---------------------------------------------------------------------------
// layout: one thread per token; warp-aggregated histograms
//   rank counts  : __ballot_sync per rank bit + popc (one smem add per warp)
//   expert counts: __match_any_sync groups equal experts (one add per group)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kLayoutThreads) layout_kernel(const int64_t* __restrict__ topk_idx, int T, int k,
                                                                 int E, int R, int32_t* __restrict__ per_rank,
                                                                 int32_t* __restrict__ per_expert,
                                                                 uint8_t* __restrict__ in_rank) {
  extern __shared__ int32_t s_hist[];  // [E + R]
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < E + R; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + tid;
  const int L = E / R;
  uint32_t mask = 0;
  const bool valid = t < T;
  for (int j = 0; j < k; ++j) {
    int64_t e = valid ? topk_idx[(size_t)t * k + j] : -1;
    if (e >= E) e = -1;  // out-of-range experts are treated as masked
    if (e >= 0) mask |= 1u << (int)(e / L);
    const unsigned peers = __match_any_sync(0xffffffffu, (unsigned long long)e);
    if (e >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_hist[e], __popc(peers));
  }
  if (valid)
    for (int d = 0; d < R; ++d) in_rank[(size_t)t * R + d] = (mask >> d) & 1u;
  for (int d = 0; d < R; ++d) {
    const unsigned b = __ballot_sync(0xffffffffu, (mask >> d) & 1u);
    if (lane == 0 && b) atomicAdd(&s_hist[E + d], __popc(b));
  }
  __syncthreads();
  for (int i = tid; i < E; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&per_expert[i], s_hist[i]);
  for (int i = tid; i < R; i += blockDim.x)
    if (s_hist[E + i]) atomicAdd(&per_rank[i], s_hist[E + i]);
}

// Inclusive scan of n <= 32*k ints in shared memory by one warp; writes the
// scanned row to `out` (global) and returns the total.
__device__ __forceinline__ int warp_inclusive_scan_row(const int32_t* in, int32_t* out, int n, int lane) {
  const int per = (n + 31) / 32, base = lane * per;
  int local = 0;
  for (int i = 0; i < per; ++i)
    if (base + i < n) local += in[base + i];
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  int run = incl - local;
  for (int i = 0; i < per; ++i) {
    if (base + i < n) {
      run += in[base + i];
      out[base + i] = run;
    }
  }
  return __shfl_sync(0xffffffffu, incl, 31);
}

// ---------------------------------------------------------------------------
// notify: one block per (local) rank.
// ---------------------------------------------------------------------------
struct NotifyParams {
  int n_local, num_channels;
  uint32_t epoch[kMaxLocal];
  RankView rv[kMaxLocal];
  epb_dispatch_args_t a[kMaxLocal];
  epb_recv_layout_t lay;
  int num_slots;
};

__global__ void __launch_bounds__(kNotifyThreads, 1) notify_kernel(const __grid_constant__ NotifyParams P) {
  const int lr = blockIdx.x;
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, C = P.num_channels, T = a.num_tokens;
  const uint32_t epoch = P.epoch[lr];
  const int par = epoch & 1;
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  Meta* my = meta_of(rv.base);
  __shared__ int32_t s_cnt[kMaxRanks][kMaxChannels];
  __shared__ int32_t s_tot[kMaxRanks];
  __shared__ int32_t s_rpm[kMaxRanks][kMaxRanks];

  // 1. my per-(destination, channel) token counts; channel c = tokens [c*Tc, (c+1)*Tc).
  //    Warp per channel, lanes over tokens, per-destination counts reduced with __reduce_add_sync.
  const int Tc = (T + C - 1) / C;
  const int nwarps = nthr >> 5;
  for (int c = warp; c < C; c += nwarps) {
    const int t0 = c * Tc, t1 = min(T, t0 + Tc);
    int n[kMaxRanks];
#pragma unroll
    for (int d = 0; d < kMaxRanks; ++d) n[d] = 0;
    for (int t = t0 + lane; t < t1; t += 32) {
      const uint8_t* row = a.is_token_in_rank + (size_t)t * R;
#pragma unroll
      for (int d = 0; d < kMaxRanks; ++d)
        if (d < R) n[d] += row[d] != 0;
    }
#pragma unroll
    for (int d = 0; d < kMaxRanks; ++d) {
      if (d < R) {
        const int tot = __reduce_add_sync(0xffffffffu, n[d]);
        if (lane == 0) s_cnt[d][c] = tot;
      }
    }
  }
  __syncthreads();
  if (warp < R) {
    const int tot = warp_inclusive_scan_row(&s_cnt[warp][0], a.channel_prefix_matrix + warp * C, C, lane);
    if (lane == 0) s_tot[warp] = tot;
  }
  __syncthreads();

  // 2. post my counts into every peer's mailbox (warp d -> peer d), then stamp the epoch.
  const int L = a.num_experts > 0 ? a.num_experts / R : 0;
  if (warp < R) {
    const int d = warp;
    Meta* pm = meta_of(rv.peer[d]);
    NotifyMsg* msg = &pm->mbox[par][me];
    for (int i = lane; i < R; i += 32) msg->counts_per_rank[i] = s_tot[i];
    if (lane == 0) {
      msg->slot = a.recv_slot;
      msg->num_tokens = T;
    }
    for (int c = lane; c < C; c += 32) msg->channel_counts[c] = s_cnt[d][c];
    if (a.num_tokens_per_expert != nullptr)
      for (int e = lane; e < L; e += 32) msg->expert_counts[e] = a.num_tokens_per_expert[d * L + e];
    fence_sys();
    __syncwarp();
    if (lane == 0) st_release_sys(&pm->mbox_flag[par][me], epoch);
  }

  // 3. wait for every source's message of this epoch
  if (tid < R) wait_geq(rv, &my->mbox_flag[par][tid], epoch, 0x100 + tid);
  __syncthreads();

  // 4. prefix sums: stage every source's counts in shared memory (parallel loads),
  //    then warp scans (no serial chains of global loads).
  for (int i = tid; i < R * C; i += nthr) s_cnt[i / C][i % C] = __ldcg(&my->mbox[par][i / C].channel_counts[i % C]);
  if (tid < R * R) s_rpm[tid / R][tid % R] = __ldcg(&my->mbox[par][tid / R].counts_per_rank[tid % R]);
  __syncthreads();
  if (warp < R) {
    warp_inclusive_scan_row(&s_cnt[warp][0], a.recv_channel_prefix_matrix + warp * C, C, lane);
  } else if (warp == R && lane < R) {
    const int d = lane;  // inclusive prefix over source rank, column d
    int run = 0;
    for (int s = 0; s < R; ++s) {
      run += s_rpm[s][d];
      s_rpm[s][d] = run;
      a.rank_prefix_matrix[s * R + d] = run;
    }
  }
  if (a.num_tokens_per_expert != nullptr) {
    const int align = max(1, a.expert_alignment);
    for (int le = tid; le < L; le += nthr) {
      int n = 0;
      for (int s = 0; s < R; ++s) n += __ldcg(&my->mbox[par][s].expert_counts[le]);
      rv.host->recv_per_expert[le] = (n + align - 1) / align * align;
    }
  }
  fence_sys();
  __syncthreads();

  // 5. plan for the dispatch kernel + host publication
  if (tid == 0) {
    Scratch* sc = scratch_of(rv.base);
    int err = 0;
    int64_t detail = 0;
    const int64_t cap = P.lay.cap_rows;
    for (int d = 0; d < R; ++d) {
      const int slot_d = __ldcg(&my->mbox[par][d].slot);
      if (slot_d < 0 || slot_d >= P.num_slots) {
        err = EPB_ERR_CONFIG;
        detail = 0x10000 + d;
      }
      sc->dst_rows[d] = reinterpret_cast<uint64_t>(rv.peer[d] + P.lay.slot0_off + (int64_t)slot_d * P.lay.slot_bytes);
      sc->row_base[d] = me > 0 ? s_rpm[me - 1][d] : 0;
      if (s_rpm[R - 1][d] > cap) {  // some destination would overflow its slot
        err = EPB_ERR_CONFIG;
        detail = ((int64_t)s_rpm[R - 1][d] << 8) | d;
      }
    }
    for (int s = 0; s < R; ++s) {  // combine staging at s holds the rows s sent
      int sent = 0;
      for (int d = 0; d < R; ++d) sent += s_rpm[s][d] - (s > 0 ? s_rpm[s - 1][d] : 0);
      if (sent > cap) {
        err = EPB_ERR_CONFIG;
        detail = ((int64_t)sent << 8) | s;
      }
    }
    sc->abort = err;
    rv.host->num_recv = s_rpm[R - 1][me];
    if (err) {
      rv.host->err_detail = detail;
      rv.host->err_code = err;
    }
    fence_sys();
    st_release_sys(const_cast<int64_t*>(&rv.host->notify_epoch), (int64_t)epoch);
  }
}

// ---------------------------------------------------------------------------
// dispatch: block = channel (contiguous token range), warp = token.
// Each row is read from HBM once (kCopyUnroll x 16 B per lane in registers)
// and stored to every destination rank that needs it (dedup per rank).
// ---------------------------------------------------------------------------
struct DispatchParams {
  int n_local, num_channels;
  uint32_t expected[kMaxLocal];
  RankView rv[kMaxLocal];
  epb_dispatch_args_t a[kMaxLocal];
  epb_recv_layout_t lay;
};

__global__ void __launch_bounds__(kDispatchThreads, 1) dispatch_kernel(const __grid_constant__ DispatchParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, C = gridDim.x, c = blockIdx.x, T = a.num_tokens;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  Scratch* sc = scratch_of(rv.base);
  extern __shared__ int32_t s_pos[];  // [Tc][R]
  __shared__ char* s_dst[kMaxRanks];
  __shared__ int32_t s_rb[kMaxRanks];
  __shared__ int s_abort;
  if (tid < R) {
    s_dst[tid] = reinterpret_cast<char*>(sc->dst_rows[tid]);
    s_rb[tid] = sc->row_base[tid];
  }
  if (tid == 0) s_abort = sc->abort;
  __syncthreads();

  const int Tc = (T + C - 1) / C;
  const int t0 = c * Tc, nt = max(0, min(T, t0 + Tc) - t0);
  if (!s_abort) {
    // positions: warp d scans destination d over the channel (ballot prefix)
    if (warp < R) {
      const int d = warp;
      int run = c > 0 ? a.channel_prefix_matrix[d * C + c - 1] : 0;
      for (int g = 0; g < nt; g += 32) {
        const int tt = g + lane;
        const bool in = tt < nt && a.is_token_in_rank[(size_t)(t0 + tt) * R + d] != 0;
        const unsigned b = __ballot_sync(0xffffffffu, in);
        const int p = in ? run + __popc(b & ((1u << lane) - 1)) : -1;
        if (tt < nt) {
          s_pos[tt * R + d] = p;
          a.send_head[(size_t)(t0 + tt) * R + d] = p;
        }
        run += __popc(b);
      }
    }
    __syncthreads();

    const size_t row_bytes = (size_t)a.hidden * a.elem_bytes;
    const int n16 = (int)(row_bytes >> 4);
    const int k = a.num_topk, S = a.num_scales;
    const int L = (a.topk_idx != nullptr && a.num_experts > 0) ? a.num_experts / R : 0;
    for (int tt = warp; tt < nt; tt += nwarps) {
      const int t = t0 + tt;
      const int4* src = reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + (size_t)t * row_bytes);
      for (int base = 0; base < n16; base += 32 * kCopyUnroll) {
        int4 v[kCopyUnroll];
#pragma unroll
        for (int u = 0; u < kCopyUnroll; ++u) {
          const int i = base + u * 32 + lane;
          if (i < n16) v[u] = ld_nc_v4(src + i);
        }
        for (int d = 0; d < R; ++d) {
          const int p = s_pos[tt * R + d];
          if (p < 0) continue;
          int4* dst = reinterpret_cast<int4*>(s_dst[d] + P.lay.off_x + (size_t)(s_rb[d] + p) * row_bytes);
#pragma unroll
          for (int u = 0; u < kCopyUnroll; ++u) {
            const int i = base + u * 32 + lane;
            if (i < n16) st_v4(dst + i, v[u]);
          }
        }
      }
      // per-row metadata: scales, mapped top-k, source index
      for (int d = 0; d < R; ++d) {
        const int p = s_pos[tt * R + d];
        if (p < 0) continue;
        const size_t row = (size_t)(s_rb[d] + p);
        char* slot = s_dst[d];
        if (a.x_scales != nullptr) {
          float* ds = reinterpret_cast<float*>(slot + P.lay.off_scales) + row * S;
          for (int i = lane; i < S; i += 32) ds[i] = a.x_scales[(size_t)t * S + i];
        }
        if (a.topk_idx != nullptr && lane < k) {
          const int64_t e = a.topk_idx[(size_t)t * k + lane];
          const int64_t le = (e >= (int64_t)d * L && e < (int64_t)(d + 1) * L) ? e - (int64_t)d * L : -1;
          reinterpret_cast<int64_t*>(slot + P.lay.off_topk_idx)[row * k + lane] = le;
          if (a.topk_weights != nullptr)
            reinterpret_cast<float*>(slot + P.lay.off_topk_w)[row * k + lane] =
                le >= 0 ? a.topk_weights[(size_t)t * k + lane] : 0.0f;
        }
        if (lane == 0) reinterpret_cast<int32_t*>(slot + P.lay.off_src_idx)[row] = t;
      }
    }
  }

  // completion: every block bumps every destination's counter for me
  fence_sys();
  __syncthreads();
  if (tid < R) red_release_sys_add(&meta_of(rv.peer[tid])->disp_done[me], 1u);
  // block 0 holds the kernel open until every source's blocks have landed here
  if (c == 0 && tid < R) wait_geq(rv, &meta_of(rv.base)->disp_done[tid], P.expected[lr], 0x200 + tid);
}

// ---------------------------------------------------------------------------
// combine: cooperative grid.  Phase A pushes each received row back into its
// source's staging at the mirror of the dispatch position; phase B (after a
// cross-rank counter barrier) reduces in fp32, ascending rank order, and
// rounds once to bf16.  Rows a rank sent to itself are read from x directly.
// ---------------------------------------------------------------------------
struct CombineParams {
  int n_local;
  uint32_t epoch[kMaxLocal];
  uint32_t expected[kMaxLocal];
  RankView rv[kMaxLocal];
  epb_combine_args_t a[kMaxLocal];
  epb_recv_layout_t lay;
};

__device__ __forceinline__ void acc_bf16x8(float* acc, const int4& v) {
  const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc[2 * i] = __fadd_rn(acc[2 * i], __uint_as_float(w[i] << 16));
    acc[2 * i + 1] = __fadd_rn(acc[2 * i + 1], __uint_as_float(w[i] & 0xffff0000u));
  }
}
__device__ __forceinline__ int4 pack_bf16x8(const float* acc) {
  int4 r;
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  r.x = (int)w[0];
  r.y = (int)w[1];
  r.z = (int)w[2];
  r.w = (int)w[3];
  return r;
}

// Sum NV bf16 rows in order into one bf16 row.  Each lane keeps NV*U 16-byte
// loads in flight (U columns per lane per step, NV*U <= 8) so a warp has
// >= 4 KB outstanding whatever the fan-in; accumulation is fp32 with one
// rounding to bf16 at the end (canonical order).
template <int NV>
__device__ __forceinline__ void reduce_rows(const int4* const* rows, int4* out, int n16, int lane) {
  constexpr int U = NV >= 8 ? 1 : 8 / NV;
  const int4* r[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) r[j] = rows[j];
  for (int base = lane; base < n16; base += 32 * U) {
    int4 v[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * u;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (i < n16) v[u][j] = ld_cg_v4(r[j] + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * u;
      if (i < n16) {
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
#pragma unroll
        for (int j = 0; j < NV; ++j) acc_bf16x8(acc, v[u][j]);
        st_na_v4(out + i, pack_bf16x8(acc));
      }
    }
  }
}

__device__ __forceinline__ void zero_row(int4* out, int n16, int lane) {
  for (int i = lane; i < n16; i += 32) st_na_v4(out + i, make_int4(0, 0, 0, 0));
}

__global__ void __launch_bounds__(kCombineThreads, 1) combine_kernel(const __grid_constant__ CombineParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_combine_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, nb = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const uint32_t epoch = P.epoch[lr];
  const int par = epoch & 1;
  __shared__ int32_t s_cnt[kMaxRanks][kMaxRanks];  // count[s][d]
  __shared__ int32_t s_excl[kMaxRanks];            // first row from s in my receive order
  __shared__ int32_t s_sendpre[kMaxRanks];         // where my rows start in s's staging
  __shared__ int32_t s_mypre[kMaxRanks];           // where d's rows start in my staging
  if (tid < R * R) {
    const int s = tid / R, d = tid % R;
    const int* rpm = a.rank_prefix_matrix;
    s_cnt[s][d] = rpm[s * R + d] - (s > 0 ? rpm[(s - 1) * R + d] : 0);
  }
  __syncthreads();
  if (tid < R) {
    const int s = tid;
    s_excl[s] = s > 0 ? a.rank_prefix_matrix[(s - 1) * R + me] : 0;
    int acc = 0;
    for (int d = 0; d < me; ++d) acc += s_cnt[s][d];
    s_sendpre[s] = acc;
    acc = 0;
    for (int d = 0; d < s; ++d) acc += s_cnt[me][d];
    s_mypre[s] = acc;
  }
  __syncthreads();

  const int H = a.hidden, k = a.num_topk;
  const size_t row_bytes = (size_t)H * 2;
  const int n16 = (int)(row_bytes >> 4);
  const bool abort = scratch_of(rv.base)->abort != 0;

  // phase A: push rows back to their sources
  const int N = a.num_recv;
  const int Jb = (N + nb - 1) / nb;
  const int j0 = b * Jb, j1 = min(N, j0 + Jb);
  if (!abort) {
    for (int j = j0 + warp; j < j1; j += nwarps) {
      int s = 0;
      while (s < R - 1 && j >= s_excl[s] + s_cnt[s][me]) ++s;
      if (s == me) continue;
      const size_t drow = (size_t)(s_sendpre[s] + (j - s_excl[s]));
      char* stage = rv.peer[s] + P.lay.comb_off[par];
      const int4* src = reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + (size_t)j * row_bytes);
      int4* dst = reinterpret_cast<int4*>(stage + drow * row_bytes);
      for (int base = 0; base < n16; base += 32 * kCopyUnroll) {
        int4 v[kCopyUnroll];
#pragma unroll
        for (int u = 0; u < kCopyUnroll; ++u) {
          const int i = base + u * 32 + lane;
          if (i < n16) v[u] = ld_nc_v4(src + i);
        }
#pragma unroll
        for (int u = 0; u < kCopyUnroll; ++u) {
          const int i = base + u * 32 + lane;
          if (i < n16) st_v4(dst + i, v[u]);
        }
      }
      if (a.topk_weights != nullptr && lane < k)
        reinterpret_cast<float*>(stage + P.lay.comb_w_off)[drow * k + lane] = a.topk_weights[(size_t)j * k + lane];
    }
  }
  fence_sys();
  __syncthreads();
  if (tid < R) red_release_sys_add(&meta_of(rv.peer[tid])->comb_done[me], 1u);
  if (tid < R) wait_geq(rv, &meta_of(rv.base)->comb_done[tid], P.expected[lr], 0x300 + tid);
  __syncthreads();
  if (abort) return;

  // phase B: reduce my tokens
  const char* my_stage = rv.base + P.lay.comb_off[par];
  const int T = a.num_tokens;
  const int Tb = (T + nb - 1) / nb;
  const int tb0 = b * Tb, tb1 = min(T, tb0 + Tb);
  for (int t = tb0 + warp; t < tb1; t += nwarps) {
    const int4* rows[kMaxRanks];
    bool self_row[kMaxRanks];
    int32_t widx[kMaxRanks];
    int nvalid = 0;
#pragma unroll
    for (int d = 0; d < kMaxRanks; ++d) {
      rows[d] = nullptr;
      self_row[d] = false;
      widx[d] = -1;
      if (d < R) {
        const int p = a.send_head[(size_t)t * R + d];
        if (p >= 0) {
          if (d == me) {
            const size_t j = (size_t)(s_excl[me] + p);
            rows[d] = reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + j * row_bytes);
            self_row[d] = true;
            widx[d] = (int32_t)j;
          } else {
            const size_t srow = (size_t)(s_mypre[d] + p);
            rows[d] = reinterpret_cast<const int4*>(my_stage + srow * row_bytes);
            widx[d] = (int32_t)srow;
          }
          ++nvalid;
        }
      }
    }
    int4* out = reinterpret_cast<int4*>(static_cast<char*>(a.combined_x) + (size_t)t * row_bytes);
    // compact the contributing rows in ascending rank order (the canonical sum order)
    const int4* cr[kMaxRanks];
    int nv = 0;
#pragma unroll
    for (int d = 0; d < kMaxRanks; ++d) {
      cr[d] = nullptr;
      if (rows[d] != nullptr) cr[nv++] = rows[d];
    }
    switch (nv) {
      case 1: reduce_rows<1>(cr, out, n16, lane); break;
      case 2: reduce_rows<2>(cr, out, n16, lane); break;
      case 3: reduce_rows<3>(cr, out, n16, lane); break;
      case 4: reduce_rows<4>(cr, out, n16, lane); break;
      case 5: reduce_rows<5>(cr, out, n16, lane); break;
      case 6: reduce_rows<6>(cr, out, n16, lane); break;
      case 7: reduce_rows<7>(cr, out, n16, lane); break;
      case 8: reduce_rows<8>(cr, out, n16, lane); break;
      default: zero_row(out, n16, lane); break;
    }
    if (a.combined_topk_weights != nullptr && lane < k) {
      float w = 0.0f;
#pragma unroll
      for (int d = 0; d < kMaxRanks; ++d) {
        if (widx[d] < 0) continue;
        const float* wsrc = self_row[d] ? a.topk_weights
                                        : reinterpret_cast<const float*>(my_stage + P.lay.comb_w_off);
        if (wsrc != nullptr) w = __fadd_rn(w, wsrc[(size_t)widx[d] * k + lane]);
      }
      a.combined_topk_weights[(size_t)t * k + lane] = w;
    }
    (void)nvalid;
  }
}

}  // namespace epb

using namespace epb;

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int compute_recv_layout(const epb_ctx* ctx, int hidden, int k, epb_recv_layout_t* L) {
  if (hidden <= 0 || hidden % 128 != 0) return epb_set_error(EPB_ERR_CONFIG, "hidden must be a positive multiple of 128");
  if (k < 0 || k > 32) return epb_set_error(EPB_ERR_CONFIG, "num_topk must be in [0, 32]");
  const size_t A = 256;
  const size_t S = (size_t)hidden / 128;
  const size_t x_row = 2 * (size_t)hidden;
  const size_t per_row = x_row + S * 4 + (size_t)k * 12 + 4;
  const size_t comb_row = 2 * (size_t)hidden + (size_t)k * 4;
  const int ns = std::max(1, ctx->cfg.num_recv_slots);
  const size_t overhead = A * (size_t)(6 * ns + 6);
  if (ctx->cfg.nvl_bytes <= overhead) return epb_set_error(EPB_ERR_CONFIG, "num_nvl_bytes too small");
  int64_t cap = (int64_t)((ctx->cfg.nvl_bytes - overhead) / (ns * per_row + 2 * comb_row));
  cap &= ~(int64_t)15;
  if (cap <= 0) return epb_set_error(EPB_ERR_CONFIG, "num_nvl_bytes too small for this hidden size");
  std::memset(L, 0, sizeof(*L));
  L->cap_rows = cap;
  L->off_x = 0;
  L->off_scales = align_up(cap * x_row, A);
  L->off_topk_idx = align_up(L->off_scales + cap * S * 4, A);
  L->off_topk_w = align_up(L->off_topk_idx + cap * (size_t)k * 8, A);
  L->off_src_idx = align_up(L->off_topk_w + cap * (size_t)k * 4, A);
  L->slot_bytes = align_up(L->off_src_idx + cap * 4, A);
  L->slot0_off = ctx->arena_off();
  const int64_t comb_bytes = align_up(cap * 2 * (size_t)hidden, A) + align_up(cap * (size_t)k * 4, A);
  L->comb_w_off = align_up(cap * 2 * (size_t)hidden, A);
  L->comb_off[0] = L->slot0_off + ns * L->slot_bytes;
  L->comb_off[1] = L->comb_off[0] + comb_bytes;
  if ((size_t)(L->comb_off[1] + comb_bytes - L->slot0_off) > ctx->cfg.nvl_bytes)
    return epb_set_error(EPB_ERR_CONFIG, "internal: recv layout exceeds arena");
  return EPB_OK;
}

extern "C" int epb_recv_layout(epb_t* ctx, int hidden, int num_topk, epb_recv_layout_t* out) {
  if (!ctx || !out) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  return compute_recv_layout(ctx, hidden, num_topk, out);
}

extern "C" int epb_get_dispatch_layout(const int64_t* topk_idx, int num_tokens, int num_topk, int num_experts,
                                       int num_ranks, int32_t* num_tokens_per_rank, int32_t* num_tokens_per_expert,
                                       uint8_t* is_token_in_rank, void* stream) {
  if (num_ranks <= 0 || num_ranks > kMaxRanks) return epb_set_error(EPB_ERR_CONFIG, "num_ranks out of range");
  if (num_experts <= 0 || num_experts % num_ranks != 0)
    return epb_set_error(EPB_ERR_CONFIG, "num_experts must be a positive multiple of num_ranks");
  if (num_topk <= 0 || num_topk > 32) return epb_set_error(EPB_ERR_CONFIG, "num_topk must be in [1, 32]");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  EPB_CUDA(cudaMemsetAsync(num_tokens_per_rank, 0, sizeof(int32_t) * num_ranks, st));
  EPB_CUDA(cudaMemsetAsync(num_tokens_per_expert, 0, sizeof(int32_t) * num_experts, st));
  if (num_tokens == 0) return EPB_OK;
  const int blocks = (num_tokens + kLayoutThreads - 1) / kLayoutThreads;
  const size_t smem = sizeof(int32_t) * (num_experts + num_ranks);
  if (smem > 48 * 1024) return epb_set_error(EPB_ERR_CONFIG, "num_experts too large for layout kernel");
  layout_kernel<<<blocks, kLayoutThreads, smem, st>>>(topk_idx, num_tokens, num_topk, num_experts, num_ranks,
                                                      num_tokens_per_rank, num_tokens_per_expert, is_token_in_rank);
  EPB_CUDA(cudaGetLastError());
  return EPB_OK;
}

static int check_group(epb_t* const* ctxs, int n) {
  if (!ctxs || n <= 0 || n > kMaxLocal) return epb_set_error(EPB_ERR_PROTOCOL, "bad local group");
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i]) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
    for (int r = 0; r < ctxs[i]->world; ++r)
      if (!ctxs[i]->peer[r]) return epb_set_error(EPB_ERR_CONNECTION, "peers not opened");
  }
  return EPB_OK;
}

extern "C" int epb_notify_dispatch(epb_t* const* ctxs, int n_local, const epb_dispatch_args_t* args,
                                   int num_channels, void* stream) {
  if (int e = check_group(ctxs, n_local)) return e;
  if (num_channels <= 0 || num_channels > kMaxChannels) return epb_set_error(EPB_ERR_CONFIG, "num_channels out of range");
  NotifyParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_local = n_local;
  P.num_channels = num_channels;
  P.num_slots = std::max(1, ctxs[0]->cfg.num_recv_slots);
  for (int i = 0; i < n_local; ++i) {
    epb_ctx* c = ctxs[i];
    const epb_dispatch_args_t& a = args[i];
    if (a.num_experts > 0 && (a.num_experts % c->world != 0 || a.num_experts / c->world > kMaxLocalExperts))
      return epb_set_error(EPB_ERR_CONFIG, "num_experts must be a multiple of world (<= 1024 local experts)");
    if (int e = compute_recv_layout(c, a.hidden, a.num_topk, &P.lay)) return e;
    P.epoch[i] = ++c->disp_epoch;
    P.rv[i] = c->view();
    P.a[i] = a;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(cudaLaunchCooperativeKernel((void*)notify_kernel, dim3(n_local), dim3(kNotifyThreads), kargs, 0, st));
  return EPB_OK;
}

extern "C" int epb_wait_notify(epb_t* ctx, int64_t* num_recv, int32_t* num_recv_per_expert, int num_local_experts,
                               double timeout_s) {
  if (!ctx) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
  const int64_t want = ctx->disp_epoch;
  auto t0 = std::chrono::steady_clock::now();
  while (true) {
    int64_t got = ctx->host->notify_epoch;
    if (got == want) break;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
      cudaError_t ce = cudaGetLastError();
      if (ce != cudaSuccess) return epb_cuda_check(ce, "notify kernel");
      return epb_set_error(EPB_ERR_DEADLOCK, "notify_dispatch timed out waiting for peers");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  if (ctx->host->err_code != 0) {
    char buf[160];
    snprintf(buf, sizeof(buf), "device reported error %lld (detail 0x%llx) in notify_dispatch",
             (long long)ctx->host->err_code, (long long)ctx->host->err_detail);
    return epb_set_error((int)ctx->host->err_code, buf);
  }
  if (num_recv) *num_recv = ctx->host->num_recv;
  if (num_recv_per_expert) {
    if (num_local_experts < 0 || num_local_experts > kMaxLocalExperts)
      return epb_set_error(EPB_ERR_PROTOCOL, "num_local_experts out of range");
    for (int i = 0; i < num_local_experts; ++i) num_recv_per_expert[i] = ctx->host->recv_per_expert[i];
  }
  return EPB_OK;
}

extern "C" int epb_dispatch(epb_t* const* ctxs, int n_local, const epb_dispatch_args_t* args, int num_channels,
                            void* stream) {
  if (int e = check_group(ctxs, n_local)) return e;
  DispatchParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_local = n_local;
  P.num_channels = num_channels;
  int max_tc = 1;
  for (int i = 0; i < n_local; ++i) {
    epb_ctx* c = ctxs[i];
    const epb_dispatch_args_t& a = args[i];
    if (a.elem_bytes != 1 && a.elem_bytes != 2) return epb_set_error(EPB_ERR_CONFIG, "elem_bytes must be 1 or 2");
    if (((size_t)a.hidden * a.elem_bytes) % 16 != 0) return epb_set_error(EPB_ERR_CONFIG, "row bytes must be 16-aligned");
    if (int e = compute_recv_layout(c, a.hidden, a.num_topk, &P.lay)) return e;
    c->disp_cum += (uint32_t)num_channels;
    P.expected[i] = c->disp_cum;
    P.rv[i] = c->view();
    P.a[i] = a;
    max_tc = std::max(max_tc, (a.num_tokens + num_channels - 1) / num_channels);
  }
  const size_t smem = sizeof(int32_t) * (size_t)max_tc * ctxs[0]->world;
  if (smem > 200 * 1024) return epb_set_error(EPB_ERR_CONFIG, "too many tokens per channel; raise num_sms");
  if (smem > 48 * 1024) EPB_CUDA(cudaFuncSetAttribute(dispatch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dispatch_kernel<<<dim3(num_channels, n_local), kDispatchThreads, smem, st>>>(P);
  EPB_CUDA(cudaGetLastError());
  return EPB_OK;
}

extern "C" int epb_combine(epb_t* const* ctxs, int n_local, const epb_combine_args_t* args, int num_sms,
                           void* stream) {
  if (int e = check_group(ctxs, n_local)) return e;
  CombineParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_local = n_local;
  int nb = std::max(1, num_sms / n_local);
  int max_active = 0;
  EPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_active, combine_kernel, kCombineThreads, 0));
  nb = std::min(nb, std::max(1, max_active * ctxs[0]->num_sms / n_local));
  for (int i = 0; i < n_local; ++i) {
    epb_ctx* c = ctxs[i];
    const epb_combine_args_t& a = args[i];
    if (int e = compute_recv_layout(c, a.hidden, a.num_topk, &P.lay)) return e;
    P.epoch[i] = ++c->comb_epoch;
    c->comb_cum += (uint32_t)nb;
    P.expected[i] = c->comb_cum;
    P.rv[i] = c->view();
    P.a[i] = a;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(cudaLaunchCooperativeKernel((void*)combine_kernel, dim3(nb, n_local), dim3(kCombineThreads), kargs, 0, st));
  return EPB_OK;
}
