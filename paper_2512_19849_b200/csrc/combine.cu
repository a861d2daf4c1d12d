// combine.cu — normal-mode combine on sm_100a (DeepEP Buffer.combine;
// SPEC.md:446-454 combine, PAPER.md:142 hierarchical reduce).
//
// One cooperative kernel: phase A pushes each received row back to its
// source rank, into the mirror of the position the source sent it from;
// a cross-rank counter barrier; phase B reduces every token's partials in
// fp32 in ascending rank order (canonical order) and rounds
// once to bf16.  Rows a rank sent to itself are read in place.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "ctx.h"
#include "ll_common.cuh"

namespace epb {

// Two instantiations (no register spills, no calls on the reduce path):
//   fan-in <= 1 (one rank: the EP=1 copy path): 16 warps, <= 128 registers;
//   fan-in <= 8 (every reducer inlined):         8 warps, <= 255 registers.
constexpr int kCombineThreadsSolo = 512;
constexpr int kCombineThreads = 256;
constexpr int kCopyUnroll = 7;
constexpr int kStreamAutoBlocks = 48;  // streamed push combine at <= this many blocks per rank
// ---------------------------------------------------------------------------
// combine: cooperative grid.  Phase A pushes each received row back into its
// source's staging at the mirror of the dispatch position; phase B (after a
// cross-rank counter barrier) reduces in fp32, ascending rank order, and
// rounds once to bf16.  Rows a rank sent to itself are read from x directly.
// ---------------------------------------------------------------------------
struct CombineParams {
  int n_local;
  int proxy;                     // ht_transport = CPU proxy: rows go back through the FIFO
  int phase;                     // proxy: 1 = stage + hand rows to the proxy, 2 = reduce
  int fifo_channels;
  uint64_t ht_calls[kMaxLocal];  // proxy transport: expected ht_sig[1][src]
  int seg16;                     // reduce work unit: 16-byte columns per (token, segment); 0 = whole rows
  int tma;                       // reduce from shared memory filled by bulk copies (small SM budgets)
  int tma_seg;                   // bytes per partial per bulk unit
  int stream;                    // streamed push (R > 1, NVLink): 1 = always, 2 = in place of a two-phase push
  int force_push;                // two-phase push even when every input lives in its region
  int push_warps;                // stream: warps per block that push (the rest reduce)
  int push_lanes;                // stream_tma: issuing lanes per push warp (each: one row buffer)
  int stream_tma;                // stream: rows pushed by bulk copies (HBM -> smem -> peer)
  int row_pad;                   // stream_tma: bytes per row buffer
  int flag_rows;                 // stream: rows per arrival word (chunk)
  int dbg;                       // stream timing decomposition (EPB_COMBINE_DEBUG): 1 no reduce, 2 no row copies
  int bump;                      // this launch ends the call: store the next epoch / done target
                                 // (device-resident, norm_call_begin/_end; the proxy's stage launch does not)
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
// Where rank d's partial of a token lives: base[d] + (row0[d] + send_head[t][d]) rows.
//   push mode: base[me] = x (my input), base[d] = my staging (rows pushed back by d)
//   pull mode: base[d] = d's input inside d's region, read over NVLink
// (kept in shared memory: it is indexed by the runtime rank id)
struct RowSrc {
  const char* base[kMaxRanks];
  const char* wbase[kMaxRanks];
  int row0[kMaxRanks];
  size_t row_bytes;
};

// += 1 on destination d's per-source counter (gpu scope suffices for myself)
__device__ __forceinline__ void bump_done(const RankView& rv, int d, int me) {
  if (d == me) red_release_gpu_add(&meta_of(rv.peer[d])->comb_done[me], 1u);
  else red_release_sys_add(&meta_of(rv.peer[d])->comb_done[me], 1u);
}

template <int NV>
__device__ __forceinline__ void reduce_rows(const RowSrc& rs, uint32_t mask, const int32_t* sh, int4* out, int i0,
                                            int n16, int lane) {
  constexpr int U = NV == 1 ? 7 : (NV >= 8 ? 1 : 8 / NV);  // NV = 1: one 224-column segment per lane pass
  const int4* r[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int d = __fns(mask, 0, j + 1);  // (j+1)-th contributing rank, ascending
    r[j] = reinterpret_cast<const int4*>(rs.base[d] + (size_t)(rs.row0[d] + sh[d]) * rs.row_bytes);
  }
#pragma unroll 1
  for (int base = i0 + lane; base < n16; base += 32 * U) {
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


__device__ __forceinline__ void zero_row(int4* out, int i0, int n16, int lane) {
  for (int i = i0 + lane; i < n16; i += 32) st_na_v4(out + i, make_int4(0, 0, 0, 0));
}

// Work unit of the reduce: a (token, row segment) pair; P.seg16 = 0 means
// whole rows (the default, measured fastest).

// Phase B: reduce my tokens.  pull: partial d is read in place from d's input
// (over NVLink); else from my staging, where the sources pushed their rows.
// send_head rows of a block's tokens, loaded at kernel entry (their latency
// overlaps the mode exchange / barrier); blocks with more tokens read global
constexpr int kShTokens = 64;

// Bulk-copy reduce (small SM budgets, where a warp's few 16-byte loads in
// flight cannot cover NVLink latency): warps [0, kCombTmaWarps) each run a
// ring of kCombTmaStages stages; a unit = (token, segment) and its stage holds
// the segment of every contributing partial, bulk-loaded (cp.async.bulk, the
// TMA engine) from the partial's row — a peer's input over NVLink (pull) or my
// staging (push) — against one mbarrier.  All 32 lanes then reduce the stage
// in fp32, ascending rank order (the canonical order, bit-identical to the
// register path), round once to bf16 and store.
constexpr int kCombTmaWarps = 4, kCombTmaStages = 3;

__device__ __noinline__ void reduce_tokens_bulk(const CombineParams& P, int lr, const RowSrc& rs,
                                               const int32_t (*s_sh)[kMaxRanks], int tb0, int tb1, bool cached) {
  const epb_combine_args_t& a = P.a[lr];
  const int R = P.rv[lr].world, k = a.num_topk;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t row_bytes = rs.row_bytes;
  const int seg = P.tma_seg, nseg = (int)((row_bytes + seg - 1) / seg);
  const int units = (tb1 - tb0) * nseg;
  __shared__ __align__(8) uint64_t s_bar[kCombTmaWarps][kCombTmaStages];
  extern __shared__ __align__(128) uint8_t s_ring[];
  // the block's send_head rows, staged once in shared memory after the rings
  // (unit bookkeeping must not wait on global loads: lane 0 issues the copies)
  int32_t* s_shb = reinterpret_cast<int32_t*>(s_ring + (size_t)kCombTmaWarps * kCombTmaStages * R * seg);
  for (int i = tid; i < (tb1 - tb0) * R; i += blockDim.x) s_shb[i] = a.send_head[(size_t)tb0 * R + i];
  __syncthreads();
  if (warp >= kCombTmaWarps) return;
  uint8_t* ring = s_ring + (size_t)warp * kCombTmaStages * R * seg;
  uint64_t* bar = s_bar[warp];
  if (lane == 0) {
    for (int st = 0; st < kCombTmaStages; ++st) mbar_init(&bar[st], 1);
    fence_async_shared();
  }
  __syncwarp();
  const int n_my = units > warp ? (units - warp + kCombTmaWarps - 1) / kCombTmaWarps : 0;
  auto unit_info = [&](int i, int& t, size_t& off, uint32_t& len, const int32_t*& sh, uint32_t& mask) {
    const int u = warp + i * kCombTmaWarps;
    t = tb0 + u / nseg;
    off = (size_t)(u % nseg) * seg;
    len = (uint32_t)min((size_t)seg, row_bytes - off);
    sh = s_shb + (size_t)(t - tb0) * R;
    mask = 0;
    for (int d = 0; d < R; ++d)
      if (sh[d] >= 0) mask |= 1u << d;
  };
  auto issue = [&](int i) {  // lane 0
    int t;
    size_t off;
    uint32_t len, mask;
    const int32_t* sh;
    unit_info(i, t, off, len, sh, mask);
    const int st = i % kCombTmaStages;
    mbar_expect_tx(&bar[st], len * (uint32_t)__popc(mask));
    int j = 0;
    for (uint32_t m = mask; m != 0; m &= m - 1, ++j) {
      const int d = __ffs(m) - 1;
      const char* src = rs.base[d] + (size_t)(rs.row0[d] + sh[d]) * row_bytes + off;
      bulk_load(ring + ((size_t)st * R + j) * seg, src, len, &bar[st]);
    }
  };
  if (lane == 0)
    for (int i = 0; i < min(n_my, kCombTmaStages); ++i) issue(i);
  for (int i = 0; i < n_my; ++i) {
    const int st = i % kCombTmaStages;
    int t;
    size_t off;
    uint32_t len, mask;
    const int32_t* sh;
    unit_info(i, t, off, len, sh, mask);
    while (!mbar_try_wait(&bar[st], (uint32_t)((i / kCombTmaStages) & 1))) {
    }
    const int nv = __popc(mask);
    const int4* stage = reinterpret_cast<const int4*>(ring + (size_t)st * R * seg);
    int4* out = reinterpret_cast<int4*>(static_cast<char*>(a.combined_x) + (size_t)t * row_bytes + off);
    const int n16 = (int)(len >> 4), s16 = seg >> 4;
    for (int c = lane; c < n16; c += 32) {
      float acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
      for (int j = 0; j < nv; ++j) acc_bf16x8(acc, stage[(size_t)j * s16 + c]);
      st_na_v4(out + c, pack_bf16x8(acc));
    }
    if (off == 0 && a.combined_topk_weights != nullptr && lane < k) {
      float w = 0.0f;
      for (uint32_t m = mask; m != 0; m &= m - 1) {
        const int d = __ffs(m) - 1;
        const float* wsrc = reinterpret_cast<const float*>(rs.wbase[d]);
        if (wsrc != nullptr) w = __fadd_rn(w, wsrc[(size_t)(rs.row0[d] + sh[d]) * k + lane]);
      }
      a.combined_topk_weights[(size_t)t * k + lane] = w;
    }
    __syncwarp();  // every lane has read the stage
    if (lane == 0 && i + kCombTmaStages < n_my) {
      fence_async_shared();  // generic-proxy reads of the stage before its async-proxy refill
      issue(i + kCombTmaStages);
    }
  }
}

template <int kMaxFan>
__device__ __forceinline__ void reduce_tokens(const CombineParams& P, int lr, bool pull, const int64_t* s_xoff,
                                              const int64_t* s_woff, const int32_t* s_excl, const int32_t* s_mypre,
                                              const int32_t (*s_sh)[kMaxRanks], int par) {
  const RankView& rv = P.rv[lr];
  const epb_combine_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, nb = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int k = a.num_topk;
  const size_t row_bytes = (size_t)a.hidden * 2;
  const int n16 = (int)(row_bytes >> 4);
  const char* my_stage = rv.base + P.lay.comb_off[par];
  const int T = a.num_tokens;
  const int Tb = (T + nb - 1) / nb;
  const int tb0 = b * Tb, tb1 = min(T, tb0 + Tb);
  __shared__ RowSrc rs;
  if (tid == 0) rs.row_bytes = row_bytes;
  if (tid < kMaxRanks) {
    const int d = tid;
    if (d == me) {
      rs.base[d] = static_cast<const char*>(a.x);
      rs.wbase[d] = reinterpret_cast<const char*>(a.topk_weights);
      rs.row0[d] = s_excl[me];
    } else if (pull) {
      rs.base[d] = d < R ? rv.peer[d] + s_xoff[d] : nullptr;
      rs.wbase[d] = (d < R && s_woff[d] >= 0) ? rv.peer[d] + s_woff[d] : nullptr;
      rs.row0[d] = (d < R && me > 0) ? a.rank_prefix_matrix[(me - 1) * R + d] : 0;  // my first row at d
    } else {
      rs.base[d] = my_stage;
      rs.wbase[d] = my_stage + P.lay.comb_w_off;
      rs.row0[d] = s_mypre[d];
    }
  }
  __syncthreads();
  const bool cached = tb1 - tb0 <= kShTokens;
  if (P.tma) {
    reduce_tokens_bulk(P, lr, rs, s_sh, tb0, tb1, cached);
    return;
  }
  const int seg16 = P.seg16 > 0 ? P.seg16 : n16;
  const int segs = (n16 + seg16 - 1) / seg16;
  for (int unit = warp; unit < (tb1 - tb0) * segs; unit += nwarps) {
    const int t = tb0 + unit / segs, sg = unit % segs;
    const int i0 = sg * seg16, i1 = min(n16, i0 + seg16);
    const int32_t* sh = cached ? s_sh[t - tb0] : a.send_head + (size_t)t * R;
    // contributing ranks as a bitmask; rows are taken in ascending rank order
    // (the canonical sum order) via __fns inside reduce_rows
    uint32_t mask = 0;
    if (lane < R && sh[lane] >= 0) mask = 1u << lane;
    mask = __reduce_or_sync(0xffffffffu, mask);
    int4* out = reinterpret_cast<int4*>(static_cast<char*>(a.combined_x) + (size_t)t * row_bytes);
    switch (__popc(mask)) {
      case 1: reduce_rows<1>(rs, mask, sh, out, i0, i1, lane); break;
      case 2: if constexpr (kMaxFan >= 2) reduce_rows<2>(rs, mask, sh, out, i0, i1, lane); break;
      case 3: if constexpr (kMaxFan >= 3) reduce_rows<3>(rs, mask, sh, out, i0, i1, lane); break;
      case 4: if constexpr (kMaxFan >= 4) reduce_rows<4>(rs, mask, sh, out, i0, i1, lane); break;
      case 5: if constexpr (kMaxFan >= 5) reduce_rows<5>(rs, mask, sh, out, i0, i1, lane); break;
      case 6: if constexpr (kMaxFan >= 6) reduce_rows<6>(rs, mask, sh, out, i0, i1, lane); break;
      case 7: if constexpr (kMaxFan >= 7) reduce_rows<7>(rs, mask, sh, out, i0, i1, lane); break;
      case 8: if constexpr (kMaxFan >= 8) reduce_rows<8>(rs, mask, sh, out, i0, i1, lane); break;
      default: zero_row(out, i0, i1, lane); break;
    }
    if (sg == 0 && a.combined_topk_weights != nullptr && lane < k) {
      float w = 0.0f;
      for (uint32_t m = mask; m != 0; m &= m - 1) {
        const int d = __ffs(m) - 1;
        const float* wsrc = reinterpret_cast<const float*>(rs.wbase[d]);
        if (wsrc != nullptr) w = __fadd_rn(w, wsrc[(size_t)(rs.row0[d] + sh[d]) * k + lane]);
      }
      a.combined_topk_weights[(size_t)t * k + lane] = w;
    }
  }
}

// Proxy transport (PAPER.md:142 hierarchical reduce, data moved by the CPU
// proxy): each source's rows are contiguous in my receive order, so one WRITE
// per source (rows, then weights) lands them at the mirror position in the
// source's staging, followed by an ATOMIC on its ht_sig[1][me].  Inputs inside
// my region are sent in place; others are first copied to my send staging.
__device__ __noinline__ void push_combine_cmds(const CombineParams& P, int lr, const int32_t (*s_cnt)[kMaxRanks],
                                               const int32_t* s_excl, const int32_t* s_sendpre, int64_t x_src,
                                               int64_t w_src, bool aborted, int par) {
  const RankView& rv = P.rv[lr];
  const epb_combine_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, k = a.num_topk;
  const int64_t arena = (int64_t)kRegionHeader, row_bytes = (int64_t)a.hidden * 2;
  for (int s = 0; s < R; ++s) {
    if (s == me) continue;
    const int ch = s % P.fifo_channels;
    const int64_t cnt = s_cnt[s][me];
    uint64_t lo, hi;
    if (!aborted && cnt > 0) {
      const int64_t dst = P.lay.comb_off[par] - arena;
      cmd_pack_dev(EPB_CMD_WRITE, s, ch, x_src + s_excl[s] * row_bytes, dst + s_sendpre[s] * row_bytes,
                   cnt * row_bytes, 0, lo, hi);
      if (fifo_push(rv, ch, lo, hi) < 0) return;
      if (w_src >= 0 && k > 0) {
        cmd_pack_dev(EPB_CMD_WRITE, s, ch, w_src + (int64_t)s_excl[s] * k * 4,
                     dst + P.lay.comb_w_off + (int64_t)s_sendpre[s] * k * 4, cnt * k * 4, 0, lo, hi);
        if (fifo_push(rv, ch, lo, hi) < 0) return;
      }
    }
    cmd_pack_dev(EPB_CMD_ATOMIC, s, ch, 0, offsetof(Meta, ht_sig) + sizeof(uint64_t) * (kMaxRanks + me), 1, 0, lo,
                 hi);
    if (fifo_push(rv, ch, lo, hi) < 0) return;
  }
}

__device__ __forceinline__ void combine_via_proxy(const CombineParams& P, int lr, const int32_t (*s_cnt)[kMaxRanks],
                                                  const int32_t* s_excl, const int32_t* s_sendpre, bool abort,
                                                  int par, uint32_t target) {
  const RankView& rv = P.rv[lr];
  const epb_combine_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, nb = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int N = a.num_recv, k = a.num_topk;
  const size_t row_bytes = (size_t)a.hidden * 2;
  const int n16 = (int)(row_bytes >> 4);
  Scratch* sc = scratch_of(rv.base);
  const char* xp = static_cast<const char*>(a.x);
  const char* wp = reinterpret_cast<const char*>(a.topk_weights);
  const char* lo = rv.base + kRegionHeader;
  const char* hi = rv.base + rv.region_bytes;
  const bool in_place = xp >= lo && xp + (size_t)N * row_bytes <= hi &&
                        (wp == nullptr || (wp >= lo && wp + (size_t)N * k * 4 <= hi));
  char* stage = rv.base + P.lay.send_off;
  if (!abort && !in_place) {
    // the previous dispatch's WRITEs read this staging: wait until the proxy
    // has completed every command pushed so far
    if (tid < P.fifo_channels) {
      const int64_t* ctl = reinterpret_cast<const int64_t*>(sc->fifo_ctl[tid]);
      const int64_t want = sc->fifo_tail[tid];
      uint64_t t0 = 0;
      while (ld_acquire_sys(ctl + EPB_CTL_COMPLETED) < want) {
        const uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > rv.timeout_ns) {
          report_error(rv, EPB_ERR_DEADLOCK, 0x340 + tid);
          break;
        }
      }
    }
    __syncthreads();
    const int Jb = (N + nb - 1) / nb;
    const int j0 = b * Jb, j1 = min(N, j0 + Jb);
    for (int j = j0 + warp; j < j1; j += nwarps) {
      int s = 0;
      while (s < R - 1 && j >= s_excl[s] + s_cnt[s][me]) ++s;
      if (s == me) continue;  // my own partials are reduced in place
      const int4* src = reinterpret_cast<const int4*>(xp + (size_t)j * row_bytes);
      int4* dst = reinterpret_cast<int4*>(stage + P.lay.off_x + (size_t)j * row_bytes);
      for (int i = lane; i < n16; i += 32) st_v4(dst + i, ld_nc_v4(src + i));
      if (wp != nullptr && lane < k)
        reinterpret_cast<float*>(stage + P.lay.off_topk_w)[(size_t)j * k + lane] = a.topk_weights[(size_t)j * k + lane];
    }
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t old = atom_add_acq_rel_gpu(&meta_of(rv.base)->comb_done[me], 1u);
    if (old + 1 == target) {  // the last of my blocks hands the rows to the proxy
      const int64_t arena = (int64_t)kRegionHeader;
      const int64_t x_src = in_place ? (int64_t)(xp - rv.base) - arena : P.lay.send_off + P.lay.off_x - arena;
      const int64_t w_src = wp == nullptr ? -1
                            : in_place ? (int64_t)(wp - rv.base) - arena
                                       : P.lay.send_off + P.lay.off_topk_w - arena;
      push_combine_cmds(P, lr, s_cnt, s_excl, s_sendpre, x_src, w_src, abort, par);
    }
  }
}

// Proxy transport, between the two combine launches: one block per local rank
// waits until every source's rows (and its ATOMIC) have landed.  The copies
// run on the proxy's streams while only these blocks are resident.
__global__ void combine_proxy_wait_kernel(const __grid_constant__ CombineParams P) {
  const RankView& rv = P.rv[blockIdx.x];
  const int tid = threadIdx.x;
  if (tid < rv.world && tid != rv.rank)
    wait_geq64(rv, &meta_of(rv.base)->ht_sig[1][tid], P.ht_calls[blockIdx.x], 0x320 + tid, 500);
}

// Streamed push combine (R > 1 over NVLink).
// Push and reduce overlap instead of running as two phases around a barrier:
//   push warps  [0, push_warps): row i of every source o (the i-th row o sent
//     me) goes back into o's staging at the mirror position, rows taken in
//     waves i = gw, gw + NW, ... with all sources in lockstep; after each row
//     lane 0 stores the call epoch into o's arrival word of that row with
//     st.release.sys (in-band completion: no counter, no barrier);
//   reduce warps: tokens t = rw, rw + NR, ... (the order the rows arrive in);
//     lane d waits for the arrival word of d's partial, then the warp reduces
//     in fp32, ascending rank order, exactly as the two-phase push mode.
// Peers only write into my staging (never read my memory), and every row a
// peer writes is awaited by one of my tokens, so no exit barrier is needed.
__device__ __forceinline__ void wait_epoch_sys(const RankView& rv, const uint32_t* p, uint32_t epoch, int64_t tag) {
  uint64_t t0 = 0;
  int iter = 0;
  while (static_cast<int32_t>(ld_acquire_sys(p) - epoch) < 0) {
    __nanosleep(64);
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

template <int kMaxFan>
__device__ __forceinline__ void combine_stream(const CombineParams& P, int lr, const int32_t (*s_cnt)[kMaxRanks],
                                               const int32_t* s_excl, const int32_t* s_sendpre,
                                               const int32_t* s_mypre, uint32_t epoch, int par) {
  const RankView& rv = P.rv[lr];
  const epb_combine_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, nb = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int k = a.num_topk, T = a.num_tokens, PW = P.push_warps;
  const size_t row_bytes = (size_t)a.hidden * 2;
  const int n16 = (int)(row_bytes >> 4);
  const char* my_stage = rv.base + P.lay.comb_off[par];
  __shared__ RowSrc rs;
  if (tid == 0) rs.row_bytes = row_bytes;
  if (tid < kMaxRanks) {
    const int d = tid;
    rs.base[d] = d == me ? static_cast<const char*>(a.x) : my_stage;
    rs.wbase[d] = d == me ? reinterpret_cast<const char*>(a.topk_weights) : my_stage + P.lay.comb_w_off;
    rs.row0[d] = d == me ? s_excl[me] : s_mypre[d];
  }
  __syncthreads();
  // rows go out in chunks of G = flag_rows consecutive rows per source; the
  // arrival word of a chunk is the one of its last row (one release per chunk:
  // a release.sys per row cost ~22 us of a 120 us push at EP=2)
  const int G = P.flag_rows;
  int nchunk = 0;
  for (int o = 0; o < R; ++o)
    if (o != me) nchunk = max(nchunk, (s_cnt[o][me] + G - 1) / G);
  if (warp < PW && P.stream_tma) {
    // bulk-copy push: each issuing lane moves whole rows HBM -> its shared
    // buffer -> the owner's staging with the TMA engine (cp.async.bulk), so
    // the reduce warps keep the SM's load/store pipeline to themselves
    const int NL = P.push_lanes;
    __shared__ __align__(8) uint64_t s_pbar[32];
    extern __shared__ __align__(128) uint8_t s_prow[];
    if (lane >= NL) return;
    const int li = warp * NL + lane;
    uint8_t* buf = s_prow + (size_t)li * P.row_pad;
    uint64_t* bar = &s_pbar[li];
    mbar_init(bar, 1);
    fence_async_shared();
    uint32_t phase = 0;
    const int gi = (b * PW + warp) * NL + lane, NI = nb * PW * NL;
    for (int c = gi; c < nchunk; c += NI) {
      for (int o = 0; o < R; ++o) {
        const int n = s_cnt[o][me], i0 = c * G, i1 = min(n, i0 + G);
        if (o == me || i0 >= n) continue;
        char* stage = rv.peer[o] + P.lay.comb_off[par];
        for (int i = i0; i < i1; ++i) {
          const size_t drow = (size_t)(s_sendpre[o] + i), srow = (size_t)(s_excl[o] + i);
          if (P.dbg != 2) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // buffer read out
            mbar_expect_tx(bar, (uint32_t)row_bytes);
            bulk_load(buf, static_cast<const char*>(a.x) + srow * row_bytes, (uint32_t)row_bytes, bar);
            while (!mbar_try_wait(bar, phase)) {
            }
            phase ^= 1;
            bulk_store(stage + drow * row_bytes, buf, (uint32_t)row_bytes);
            bulk_commit();
          }
          if (a.topk_weights != nullptr)
            for (int q = 0; q < k; ++q)
              reinterpret_cast<float*>(stage + P.lay.comb_w_off)[drow * k + q] = a.topk_weights[srow * k + q];
        }
        bulk_wait_all();  // the chunk's rows are written before its arrival word
        if (P.dbg != 3)
          st_release_sys(reinterpret_cast<uint32_t*>(stage + P.lay.comb_flag_off) + s_sendpre[o] + i1 - 1, epoch);
      }
    }
    return;
  }
  if (warp < PW) {
    const int gw = b * PW + warp, NW = nb * PW;
    for (int c = gw; c < nchunk; c += NW) {
      for (int o = 0; o < R; ++o) {
        const int n = s_cnt[o][me], i0 = c * G, i1 = min(n, i0 + G);
        if (o == me || i0 >= n) continue;
        char* stage = rv.peer[o] + P.lay.comb_off[par];
        for (int i = i0; i < i1; ++i) {
          const size_t drow = (size_t)(s_sendpre[o] + i);
          const int4* src =
              reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + (size_t)(s_excl[o] + i) * row_bytes);
          int4* dst = reinterpret_cast<int4*>(stage + drow * row_bytes);
          for (int base = 0; base < n16; base += 32 * kCopyUnroll) {
            int4 v[kCopyUnroll];
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u) {
              const int cc = base + u * 32 + lane;
              if (cc < n16) v[u] = ld_nc_v4(src + cc);
            }
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u) {
              const int cc = base + u * 32 + lane;
              if (cc < n16) st_v4(dst + cc, v[u]);
            }
          }
          if (a.topk_weights != nullptr && lane < k)
            reinterpret_cast<float*>(stage + P.lay.comb_w_off)[drow * k + lane] =
                a.topk_weights[(size_t)(s_excl[o] + i) * k + lane];
        }
        __syncwarp();
        if (lane == 0 && P.dbg != 3)
          st_release_sys(reinterpret_cast<uint32_t*>(stage + P.lay.comb_flag_off) + s_sendpre[o] + i1 - 1, epoch);
      }
    }
    return;
  }
  const int RW = nwarps - PW, rw = b * RW + (warp - PW), NR = nb * RW;
  const uint32_t* my_flags = reinterpret_cast<const uint32_t*>(my_stage + P.lay.comb_flag_off);
  if (P.dbg == 3) return;
  for (int t = rw; t < T; t += NR) {
    const int32_t* sh = a.send_head + (size_t)t * R;
    const int shl = lane < R ? sh[lane] : -1;
    const uint32_t mask = __ballot_sync(0xffffffffu, shl >= 0);
    if (shl >= 0 && lane != me)  // the arrival word of the chunk holding row shl
      wait_epoch_sys(rv, my_flags + s_mypre[lane] + min(s_cnt[me][lane], (shl / G + 1) * G) - 1, epoch, 0x3c0 + lane);
    __syncwarp();
    int4* out = reinterpret_cast<int4*>(static_cast<char*>(a.combined_x) + (size_t)t * row_bytes);
    if (P.dbg == 1) continue;
    switch (__popc(mask)) {
      case 1: reduce_rows<1>(rs, mask, sh, out, 0, n16, lane); break;
      case 2: if constexpr (kMaxFan >= 2) reduce_rows<2>(rs, mask, sh, out, 0, n16, lane); break;
      case 3: if constexpr (kMaxFan >= 3) reduce_rows<3>(rs, mask, sh, out, 0, n16, lane); break;
      case 4: if constexpr (kMaxFan >= 4) reduce_rows<4>(rs, mask, sh, out, 0, n16, lane); break;
      case 5: if constexpr (kMaxFan >= 5) reduce_rows<5>(rs, mask, sh, out, 0, n16, lane); break;
      case 6: if constexpr (kMaxFan >= 6) reduce_rows<6>(rs, mask, sh, out, 0, n16, lane); break;
      case 7: if constexpr (kMaxFan >= 7) reduce_rows<7>(rs, mask, sh, out, 0, n16, lane); break;
      case 8: if constexpr (kMaxFan >= 8) reduce_rows<8>(rs, mask, sh, out, 0, n16, lane); break;
      default: zero_row(out, 0, n16, lane); break;
    }
    if (a.combined_topk_weights != nullptr && lane < k) {
      float w = 0.0f;
      for (uint32_t m = mask; m != 0; m &= m - 1) {
        const int d = __ffs(m) - 1;
        const float* wsrc = reinterpret_cast<const float*>(rs.wbase[d]);
        if (wsrc != nullptr) w = __fadd_rn(w, wsrc[(size_t)(rs.row0[d] + sh[d]) * k + lane]);
      }
      a.combined_topk_weights[(size_t)t * k + lane] = w;
    }
  }
}

template <int kMaxFan>
__device__ __forceinline__ void combine_body(const CombineParams& P, uint32_t epoch, uint32_t target) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_combine_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, nb = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int par = epoch & 1;
  trace_mark(rv, 15);
  __shared__ int32_t s_sh[kShTokens][kMaxRanks];
  {
    const int T = a.num_tokens, Tb = (T + nb - 1) / nb, tb0 = b * Tb, nt = min(T, tb0 + Tb) - tb0;
    if (nt > 0 && nt <= kShTokens)
      for (int i = threadIdx.x; i < nt * R; i += blockDim.x) s_sh[i / R][i % R] = a.send_head[(size_t)tb0 * R + i];
  }
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
  trace_mark(rv, 16);

  if constexpr (kMaxFan > 1) {  // (the one-rank instantiation never streams)
    if (P.stream == 1 && R > 1 && !abort) {
      combine_stream<kMaxFan>(P, lr, s_cnt, s_excl, s_sendpre, s_mypre, epoch, par);
      trace_mark(rv, 19);
      trace_mark_max(rv, 20);
      __syncthreads();
      if (tid < R) bump_done(rv, tid, me);  // keeps the cumulative done counters in step (no wait)
      return;
    }
  }
  // mode exchange: if every rank's combine input (and weights) lives inside its
  // symmetric region — e.g. the zero-copy recv_x of the dispatch — tokens are
  // reduced by reading the partials in place over NVLink (pull), with no push
  // and no staging pass; otherwise rows are pushed back into staging first.
  const int N = a.num_recv;
  __shared__ int64_t s_xoff[kMaxRanks], s_woff[kMaxRanks];
  if (P.proxy) {  // proxy transport: no SM access to peers' memory at all
    if (P.phase == 1) {
      combine_via_proxy(P, lr, s_cnt, s_excl, s_sendpre, abort, par, target);
      trace_mark(rv, 17);
    } else if (!abort) {
      trace_mark_max(rv, 21);
      reduce_tokens<kMaxFan>(P, lr, false, s_xoff, s_woff, s_excl, s_mypre, s_sh, par);
      trace_mark(rv, 19);
      trace_mark_max(rv, 20);
    }
    return;
  }
  if (R == 1) {  // single rank: my own input is read in place in either mode
    if (tid == 0) s_xoff[0] = 0;
  } else if (b == 0 && tid < R) {  // my offsets to every peer: tagged words (16-byte / 4-byte units)
    const char* xp = static_cast<const char*>(a.x);
    const char* wp = reinterpret_cast<const char*>(a.topk_weights);
    const char* lo = rv.base;
    const char* hi = rv.base + rv.region_bytes;
    const bool xin = xp >= lo && xp + (size_t)N * row_bytes <= hi && ((xp - lo) & 15) == 0 && (xp - lo) / 16 < kNotifyAbort;
    const bool win = wp == nullptr || (wp >= lo && wp + (size_t)N * k * 4 <= hi && ((wp - lo) & 3) == 0 &&
                                       (wp - lo) / 4 < kNotifyAbort);
    const uint32_t xo = (xin && win) ? (uint32_t)((xp - lo) / 16) : kNotifyAbort;
    const uint32_t wo = (xin && win && wp != nullptr) ? (uint32_t)((wp - lo) / 4) : kNotifyAbort;
    uint64_t* m = meta_of(rv.peer[tid])->comb_msg[par][me];
    st_relaxed_sys(&m[0], tagged(xo, epoch));
    st_relaxed_sys(&m[1], tagged(wo, epoch));
  }
  if (tid < 2 * R && R > 1) {
    const int s = tid >> 1, f = tid & 1;
    const uint32_t v = wait_tagged(rv, &meta_of(rv.base)->comb_msg[par][s][f], epoch, 0x380 + s);
    const int64_t off = v == kNotifyAbort ? -1 : (int64_t)v * (f ? 4 : 16);
    if (f) s_woff[s] = off;
    else s_xoff[s] = off;
  }
  __syncthreads();
  bool pull = !P.force_push;
  for (int d = 0; d < R; ++d) pull = pull && s_xoff[d] >= 0;
  if constexpr (kMaxFan > 1) {
    if (!pull && !abort && P.stream == 2) {  // some input outside its region: streamed push
      combine_stream<kMaxFan>(P, lr, s_cnt, s_excl, s_sendpre, s_mypre, epoch, par);
      trace_mark(rv, 19);
      trace_mark_max(rv, 20);
      __syncthreads();
      if (tid < R) bump_done(rv, tid, me);
      return;
    }
  }

  // phase A (push mode): push rows back to their sources
  const int Jb = (N + nb - 1) / nb;
  const int j0 = b * Jb, j1 = min(N, j0 + Jb);
  if (!abort && !pull) {
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
  __syncthreads();
  trace_mark(rv, 17);
  // push mode: every source's rows have landed in my staging before I reduce.
  // pull mode: the same counters are bumped after phase B instead, and mean
  // "I have finished reading your input" — no rank returns (and lets its
  // caller reuse the input) while a peer may still be reading it.
  if (!pull || abort) {
    if (tid < R) bump_done(rv, tid, me);
    if (tid < R) wait_geq(rv, &meta_of(rv.base)->comb_done[tid], target, 0x300 + tid);
    __syncthreads();
  }
  trace_mark(rv, 18);
  trace_mark_max(rv, 21);
  if (abort) return;

  reduce_tokens<kMaxFan>(P, lr, pull, s_xoff, s_woff, s_excl, s_mypre, s_sh, par);
  trace_mark(rv, 19);
  trace_mark_max(rv, 20);
  if (pull) {
    __syncthreads();  // this block's reads of the peers' inputs are complete
    if (R == 1) {     // no peer reads my input: only keep the counter in step
      if (tid == 0) atomicAdd(&meta_of(rv.base)->comb_done[0], 1u);
    } else {
      if (tid < R) bump_done(rv, tid, me);
      if (b == 0 && tid < R) wait_geq(rv, &meta_of(rv.base)->comb_done[tid], target, 0x300 + tid);
    }
  }
}

template <int kMaxFan, int kThreads>
__global__ void __launch_bounds__(kThreads, 1) combine_kernel(const __grid_constant__ CombineParams P) {
  __shared__ uint32_t s_epoch, s_target;
  if (threadIdx.x == 0) norm_call_begin(P.rv[blockIdx.y], 1, gridDim.x, &s_epoch, &s_target);
  __syncthreads();
  const uint32_t epoch = s_epoch, target = s_target;
  combine_body<kMaxFan>(P, epoch, target);
  if (threadIdx.x == 0 && P.bump) norm_call_end(P.rv[blockIdx.y], 1, epoch, target);
}

}  // namespace epb

using namespace epb;

extern "C" int epb_combine(epb_t* const* ctxs, int n_local, const epb_combine_args_t* args, int num_sms,
                           void* stream) {
  if (int e = check_group(ctxs, n_local)) return e;
  CombineParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_local = n_local;
  P.proxy = ctxs[0]->cfg.ht_transport == EPB_HT_PROXY ? 1 : 0;
  if (ctxs[0]->cfg.ht_transport == EPB_HT_RING)
    return epb_set_error(EPB_ERR_CONFIG, "ht_transport=ring: use epb_ring_combine");
  P.fifo_channels = ctxs[0]->cfg.fifo_channels;
  for (int i = 0; i < n_local; ++i)
    if (P.proxy && (ctxs[i]->cfg.fifo_channels <= 0 || !ctxs[i]->proxy || ctxs[i]->cfg.ht_transport != EPB_HT_PROXY))
      return epb_set_error(EPB_ERR_CONFIG, "ht_transport=proxy needs FIFO channels and a running proxy on every rank");
  int nb = std::max(1, num_sms / n_local);
  // one rank (EP=1): every token has fan-in 1 -> the 12-warp copy instantiation
  const bool solo = ctxs[0]->world == 1;
  const void* kern = solo ? (const void*)combine_kernel<1, kCombineThreadsSolo> : (const void*)combine_kernel<8, kCombineThreads>;
  const int threads = solo ? kCombineThreadsSolo : kCombineThreads;
  // reduce work unit: whole rows (3.5 KB row segments measured slower: EP=2 135
  // against 124 us, EP=1 22.6 against 21.8 us per combine; profiles/r02_summary.md).
  // EPB_COMBINE_SEG16 = 16-byte columns per segment (measurement knob).
  static const int seg_env = [] {
    const char* v = std::getenv("EPB_COMBINE_SEG16");
    return v ? std::atoi(v) : -1;
  }();
  P.seg16 = seg_env >= 0 ? seg_env : 0;
  // streamed push (combine_stream) for R > 1 over NVLink.  Auto (EPB_COMBINE_MODE
  // unset): always on small SM budgets (<= kStreamAutoBlocks blocks per rank: 252
  // against 500 us at 20 SMs at EP=2, 558 against 1044 us at EP=4) and, at EP=2
  // only, in place of the two-phase push when some input lives outside its region
  // (134 against 148 us; at EP=4 520 against 332 us).  With every input in its
  // region at full width the pull reduce stays (EP=2 119 against 127 us, EP=4 286
  // against 444 us; profiles/r02_combine_stream_n2.txt, r02_combine_stream_n4.txt).  EPB_COMBINE_MODE=stream | classic | push
  // forces stream / never stream / the two-phase push.  EPB_COMBINE_PUSH_WARPS = push warps per block
  static const int mode_env = [] {
    const char* v = std::getenv("EPB_COMBINE_MODE");
    if (!v) return -1;
    return std::strcmp(v, "stream") == 0 ? 1 : std::strcmp(v, "push") == 0 ? 2 : 0;
  }();
  static const int pw_env = [] {
    const char* v = std::getenv("EPB_COMBINE_PUSH_WARPS");
    return v ? std::atoi(v) : 1;
  }();
  P.stream = 0;
  if (!P.proxy && ctxs[0]->world > 1) {
    if (mode_env == 1) P.stream = 1;
    else if (mode_env < 0) P.stream = nb <= kStreamAutoBlocks ? 1 : ctxs[0]->world == 2 ? 2 : 0;
  }
  P.force_push = mode_env == 2 ? 1 : 0;
  P.push_warps = std::max(1, std::min(threads / 32 - 1, pw_env));
  // stream: bulk-copy pushers (EPB_COMBINE_STREAM_TMA=0 off; EPB_COMBINE_PUSH_LANES
  // issuing lanes per push warp, each with one row buffer in shared memory)
  static const int stma_env = [] {
    const char* v = std::getenv("EPB_COMBINE_STREAM_TMA");
    return v ? std::atoi(v) : 1;
  }();
  static const int pl_env = [] {
    const char* v = std::getenv("EPB_COMBINE_PUSH_LANES");
    return v ? std::atoi(v) : 8;
  }();
  static const int dbg_env = [] {
    const char* v = std::getenv("EPB_COMBINE_DEBUG");
    return v ? std::atoi(v) : 0;
  }();
  P.dbg = dbg_env;
  static const int fr_env = [] {
    const char* v = std::getenv("EPB_COMBINE_FLAG_ROWS");
    return v ? std::atoi(v) : 2;
  }();
  P.flag_rows = std::max(1, fr_env);
  size_t stream_smem = 0;
  if (P.stream && stma_env > 0) {
    const size_t rb = (size_t)args[0].hidden * 2;
    bool ok = rb % 16 == 0;
    for (int i = 0; i < n_local && ok; ++i)
      ok = (size_t)args[i].hidden * 2 == rb && (reinterpret_cast<uintptr_t>(args[i].x) & 15) == 0;
    P.push_lanes = std::max(1, std::min(32 / P.push_warps, pl_env));
    P.row_pad = (int)((rb + 127) & ~(size_t)127);
    stream_smem = (size_t)P.push_warps * P.push_lanes * P.row_pad;
    if (ok && stream_smem <= 200 * 1024) {
      P.stream_tma = 1;
      EPB_CUDA(epb_ensure_smem(kern, stream_smem));
    } else {
      stream_smem = 0;
    }
  }
  // bulk-copy reduce: opt-in only (EPB_TMA=1).  Parity-green, but measured slower
  // than the register path at every SM budget (N=1, 20/24/48 SMs: 280/239/124 us
  // against 76/66/38 us; profiles/r02_tma_ab_n1.txt): 4 warps x 3 stages of
  // segments in flight per block cannot match 16 warps of 16-byte loads.
  static const int tma_env = [] {
    const char* v = std::getenv("EPB_TMA");
    return v ? std::atoi(v) : -1;
  }();
  size_t smem = 0;
  if (tma_env > 0 && !P.proxy) {
    const int R = ctxs[0]->world;
    const size_t rb = (size_t)args[0].hidden * 2;
    int seg = (int)std::min<size_t>(8192, 16384 / (size_t)R) & ~15;
    seg = (int)std::min<size_t>((size_t)seg, rb);
    int tmax = 0;
    for (int i = 0; i < n_local; ++i) tmax = std::max(tmax, args[i].num_tokens);
    // rings + the send_head cache of a block's tokens (nb only shrinks below, by
    // co-residency, which 1 block/SM with <= 200 KB keeps)
    const size_t need = (size_t)kCombTmaWarps * kCombTmaStages * R * seg + (size_t)((tmax + nb - 1) / nb) * R * 4;
    bool ok = (rb % 16) == 0 && need <= 200 * 1024 && nb <= ctxs[0]->num_sms / n_local;
    for (int i = 0; i < n_local && ok; ++i) ok = (size_t)args[i].hidden * 2 == rb;
    if (ok) {
      P.tma = 1;
      P.tma_seg = seg;
      smem = need;
      EPB_CUDA(epb_ensure_smem(kern, smem));
    }
  }
  smem = std::max(smem, stream_smem);
  const int max_active = epb_max_active_blocks(kern, threads, smem);
  nb = std::min(nb, std::max(1, max_active * ctxs[0]->num_sms / n_local));
  for (int i = 0; i < n_local; ++i) {
    epb_ctx* c = ctxs[i];
    const epb_combine_args_t& a = args[i];
    if (int e = compute_recv_layout(c, a.hidden, a.num_topk, &P.lay)) return e;
    if (P.proxy) P.ht_calls[i] = ++c->ht_comb_calls;
    P.rv[i] = c->view();
    P.a[i] = a;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  if (P.proxy) {  // stage + push | wait for the peers' rows | reduce
    P.phase = 1;
    P.bump = 0;
    EPB_CUDA(cudaLaunchKernel(kern, dim3(nb, n_local), dim3(threads), kargs, 0, st));
    combine_proxy_wait_kernel<<<n_local, 32, 0, st>>>(P);
    EPB_CUDA(cudaGetLastError());
    if (std::getenv("EPB_PROXY_SYNC")) EPB_CUDA(cudaStreamSynchronize(st));  // see epb_dispatch
    P.phase = 2;
    P.bump = 1;
    EPB_CUDA(cudaLaunchKernel(kern, dim3(nb, n_local), dim3(threads), kargs, 0, st));
    return EPB_OK;
  }
  P.bump = 1;
  EPB_CUDA(epb_launch_grid_sync(kern, dim3(nb, n_local), dim3(threads), kargs, smem, st));
  return EPB_OK;
}

// Load this file's kernels now (see epb_preload_kernels, api.cpp).
cudaError_t epb_preload_combine() {
  cudaFuncAttributes attr;
  for (const void* fn : {(const void*)combine_proxy_wait_kernel, (const void*)combine_kernel<1, kCombineThreadsSolo>, (const void*)combine_kernel<8, kCombineThreads>})
    if (cudaError_t e = cudaFuncGetAttributes(&attr, fn)) return e;
  return cudaSuccess;
}
