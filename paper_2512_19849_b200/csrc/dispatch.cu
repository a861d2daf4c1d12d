// dispatch.cu — normal-mode (high-throughput) dispatch on sm_100a, one
// cooperative kernel per call:
//
//   1. every block = one channel (a contiguous token range); warp d ballots
//      the channel's tokens for destination d -> positions + per-channel count
//   2. block 0 runs the count exchange ("notify"): gathers every channel's
//      counts, posts one mailbox message per peer over NVLink (per-rank totals,
//      my receive slot, per-channel counts, per-expert counts), reads every
//      peer's message, derives the rank prefix matrix and this rank's plan
//      (destination slot + first row per destination); its first warps then
//      publish the receive counts to the host (pinned memory) for the caller's
//      tensor shapes.  Every control word on this path is a tagged word
//      (common.cuh), so there is no grid barrier, no flag and no fence: each
//      block polls exactly the words it needs.
//   3. all blocks push every deduplicated row straight into its final row of
//      the destination's receive slot: one HBM read per row, one 16-byte store
//      per lane per destination (NVLink for peers)
//   4. every block release-adds each destination's done counter; block 0 of
//      every rank holds the kernel open until all sources have landed here.
//
// Semantics: dedup per destination rank;
// receive order = (source rank, source token) — the order the reference's
// HT delivery produces (tests/golden/ht_dispatch.npz).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "ctx.h"
#include "ll_common.cuh"

namespace epb {

constexpr int kDispatchThreads = 512;
constexpr int kCopyUnroll = 7;
// Bulk-copy (TMA) path: kTmaWarps warps per block each drive a ring of
// kTmaStages units of <= 8 KB through shared memory (global -> shared bulk
// load with an mbarrier, shared -> global bulk store per destination).
constexpr int kTmaWarps = 6, kTmaStages = 4, kTmaSegMax = 8192;
constexpr int kTmaAutoChannels = 48;  // bulk copies by default at <= 48 channels (SM budgets)  // 7 x 16 B per lane in flight = 3.5 KB per warp

// Inclusive/exclusive scan of n <= 32*k ints in shared memory by one warp;
// writes the inclusive row to `incl_out` and the exclusive row to
// `excl_out` (either may be null); returns the total.
__device__ __forceinline__ int warp_scan_row(const int32_t* in, int32_t* incl_out, int32_t* excl_out, int n,
                                             int lane) {
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
      if (excl_out) excl_out[base + i] = run;
      run += in[base + i];
      if (incl_out) incl_out[base + i] = run;
    }
  }
  return __shfl_sync(0xffffffffu, incl, 31);
}

struct DispatchParams {
  int n_local, num_slots;
  int proxy;                    // ht_transport = CPU proxy (rows to peers go through the FIFO)
  int notify_only;              // chunked-ring transport: counts, handle and host counts only (chunked.cu moves rows)
  int perblock;                 // R > 1, direct transport: blocks other than 0 read the peers' mailbox
                                // words and derive their channel offsets themselves (no block-0 plan hop)
  int solo;                     // one rank, direct transport, T <= capacity: block 0 only runs the count
                                // exchange (its channel is empty) and every other block derives its own
                                // channel offset, so copies start without waiting for the plan
  int fifo_channels;
  int tma;                      // rows move through per-warp shared-memory rings with bulk copies
  int tma_seg;                  // bytes per bulk unit (a row, or a part of it)
  int tma_smem_off;             // byte offset of the rings in dynamic shared memory
  uint64_t ht_calls[kMaxLocal];  // proxy transport: expected ht_sig[0][src] (calls so far)
  uint32_t host_seq[kMaxLocal];  // tag of this call's host words (the host's call counter); the
                                 // mailbox epoch and done targets are device-resident (norm_call_begin)
  RankView rv[kMaxLocal];
  epb_dispatch_args_t a[kMaxLocal];
  epb_recv_layout_t lay;
};

// Block 0, warp R + d, at kernel start: my tokens for each of peer d's local
// experts (known from the inputs alone, so they travel while the channels are
// being counted; only the peer's host publication needs them).
__device__ __forceinline__ void post_expert_counts(const DispatchParams& P, int lr, int d, uint32_t epoch) {
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, lane = threadIdx.x & 31;
  NotifyMsg* msg = &meta_of(rv.peer[d])->mbox[epoch & 1][me];
  const int L = a.num_experts > 0 ? a.num_experts / R : 0;
  for (int base = 0; base < L; base += 32 * 8) {  // 8 loads in flight per lane, then the stores
    int v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = base + j * 32 + lane;
      v[j] = (e < L && a.num_tokens_per_expert != nullptr) ? __ldg(&a.num_tokens_per_expert[d * L + e]) : 0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = base + j * 32 + lane;
      if (e < L) st_relaxed_sys(&msg->expert_counts[e], tagged((uint32_t)v[j], epoch));
    }
  }
}

// Block 0, warps [0, kPublishWarps): the per-expert receive counts for the host
// (tagged words, HostInfo), then the receive channel prefix (handle output), while
// block 0's other warps already copy rows.  All of a thread's words are
// loaded before any is checked (one round trip when they have all arrived).
constexpr int kPublishWarps = 2;
__device__ __forceinline__ void publish_counts(const DispatchParams& P, int lr, int C, bool aborted, uint32_t epoch) {
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world;
  const int par = epoch & 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int nthr = kPublishWarps * 32;
  const Meta* my = meta_of(rv.base);
  if (aborted) return;
  const int L = a.num_experts > 0 ? a.num_experts / R : 0;
  const int align = max(1, a.expert_alignment);
  for (int le0 = tid; le0 < L; le0 += 2 * nthr) {
    uint64_t v[2][kMaxRanks];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int s = 0; s < kMaxRanks; ++s) {
        const int le = le0 + j * nthr;
        v[j][s] = (s < R && le < L) ? ld_relaxed_sys(&my->mbox[par][s].expert_counts[le]) : tagged(0, epoch);
      }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int le = le0 + j * nthr;
      if (le >= L) break;
      int n = 0;
#pragma unroll
      for (int s = 0; s < kMaxRanks; ++s)
        if (s < R)
          n += (uint32_t)v[j][s] == epoch ? (int)(v[j][s] >> 32)
                                        : (int)wait_tagged(rv, &my->mbox[par][s].expert_counts[le], epoch, 0x140 + s);
      n = (n + align - 1) / align * align;
      st_relaxed_sys(&rv.host->notify[1 + le], tagged((uint32_t)n, P.host_seq[lr]));
    }
  }
  // every source's per-channel counts -> receive channel prefix (handle output)
  constexpr int kChunks = kMaxChannels / 32;
  for (int s = warp; s < R; s += kPublishWarps) {
    uint64_t v[kChunks];
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
      const int cc = q * 32 + lane;
      v[q] = cc < C ? ld_relaxed_sys(&my->mbox[par][s].channel_counts[cc]) : tagged(0, epoch);
    }
    int run = 0;
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
      if (q * 32 >= C) break;
      const int cc = q * 32 + lane;
      const int x = (uint32_t)v[q] == epoch ? (int)(v[q] >> 32)
                                            : (int)wait_tagged(rv, &my->mbox[par][s].channel_counts[cc], epoch, 0x160 + s);
      int incl = x;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += u;
      }
      if (cc < C) a.recv_channel_prefix_matrix[s * C + cc] = run + incl;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  trace_mark(rv, 6);
}

// Block 0: gather every channel's counts (tagged words), post my counts to the
// peers, read theirs, and publish the plan (tagged words) for the other
// blocks.  After the gather only warp 0 is on the critical path (peer
// messages -> plan); the other warps publish the per-channel words meanwhile.
__device__ __forceinline__ void exchange_counts(const DispatchParams& P, int lr, int C, int32_t (*s_cnt)[kMaxChannels],
                                             int32_t (*s_rpm)[kMaxRanks], int32_t* s_slot, int* s_abort,
                                             uint32_t epoch) {
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank;
  const int par = epoch & 1;
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  Scratch* sc = scratch_of(rv.base);
  const Meta* my = meta_of(rv.base);
  trace_mark(rv, 2);
  {
    constexpr int kPer = kMaxRanks * kMaxChannels / kDispatchThreads;
    uint64_t v[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + j * nthr;
      v[j] = i < R * C ? ld_relaxed_sys(&sc->ch_cnt[i / C][i % C]) : tagged(0, epoch);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + j * nthr;
      if (i < R * C) {
        const uint32_t x = (uint32_t)v[j] == epoch ? (uint32_t)(v[j] >> 32)
                                                   : wait_tagged(rv, &sc->ch_cnt[i / C][i % C], epoch, 0x180);
        if (x == kNotifyAbort) *s_abort = EPB_ERR_DEADLOCK;
        s_cnt[i / C][i % C] = (int)x;
      }
    }
  }
  __syncthreads();
  trace_mark(rv, 1);
  if (R == 1 && warp == 0) {
    // single rank: no mailbox round trip — my totals and slot are the plan's inputs
    int s = 0;
    for (int cc = lane; cc < C; cc += 32) s += s_cnt[0][cc];
    s = __reduce_add_sync(0xffffffffu, s);
    if (lane == 0) {
      s_rpm[0][0] = s;
      s_slot[0] = a.recv_slot;
    }
  } else if (warp < R) {
    // what peer d's plan needs: my per-rank totals and my receive slot
    const int d = warp;
    NotifyMsg* msg = &meta_of(rv.peer[d])->mbox[par][me];
    for (int i = 0; i < R; ++i) {
      int s = 0;
      for (int cc = lane; cc < C; cc += 32) s += s_cnt[i][cc];
      s = __reduce_add_sync(0xffffffffu, s);
      if (lane == i) st_relaxed_sys(&msg->counts_per_rank[i], tagged((uint32_t)s, epoch));
    }
    if (lane == 31) st_relaxed_sys(&msg->slot, tagged((uint32_t)a.recv_slot, epoch));
  } else if (warp < 2 * R) {
    // each channel's offset inside my run to d (for my other blocks), the
    // per-channel counts for peer d's handle, my channel prefix matrix row d
    const int d = warp - R;
    int run = 0;
    for (int base = 0; base < C; base += 32) {
      const int cc = base + lane;
      const int v = cc < C ? s_cnt[d][cc] : 0;
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += u;
      }
      if (cc < C) st_relaxed_sys(&sc->ch_excl[d][cc], tagged((uint32_t)(run + incl - v), epoch));
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    NotifyMsg* msg = &meta_of(rv.peer[d])->mbox[par][me];
    for (int cc = lane; cc < C; cc += 32)
      st_relaxed_sys(&msg->channel_counts[cc], tagged((uint32_t)s_cnt[d][cc], epoch));
    warp_scan_row(&s_cnt[d][0], a.channel_prefix_matrix + d * C, nullptr, C, lane);
  }
  trace_mark(rv, 3);
  if (warp != 0) return;

  // warp 0: every source's totals and receive slot (<= 72 words, 3 per lane)
  constexpr int kPer = (kMaxRanks * (kMaxRanks + 1) + 31) / 32;
  uint64_t v[kPer];
#pragma unroll
  for (int j = 0; j < kPer && R > 1; ++j) {
    const int i = lane + 32 * j, s = i / (R + 1), f = i % (R + 1);
    v[j] = i < R * (R + 1) ? ld_relaxed_sys(f < R ? &my->mbox[par][s].counts_per_rank[f] : &my->mbox[par][s].slot)
                           : tagged(0, epoch);
  }
#pragma unroll
  for (int j = 0; j < kPer && R > 1; ++j) {
    const int i = lane + 32 * j, s = i / (R + 1), f = i % (R + 1);
    if (i < R * (R + 1)) {
      const uint64_t* w = f < R ? &my->mbox[par][s].counts_per_rank[f] : &my->mbox[par][s].slot;
      const uint32_t x = (uint32_t)v[j] == epoch ? (uint32_t)(v[j] >> 32) : wait_tagged(rv, w, epoch, 0x100 + s);
      if (x == kNotifyAbort) *s_abort = EPB_ERR_DEADLOCK;
      if (f < R) s_rpm[s][f] = (int)x;
      else s_slot[s] = (int)x;
    }
  }
  __syncwarp();
  trace_mark(rv, 4);
  if (lane < R) {  // inclusive prefix over source rank, column d
    int run = 0;
    for (int s = 0; s < R; ++s) {
      run += s_rpm[s][lane];
      s_rpm[s][lane] = run;
    }
  }
  __syncwarp();
  if (lane == 0 && *s_abort == 0 && !P.notify_only) {
    // capacity checks (every rank sees the same matrix, so all abort together)
    int err = 0;
    int64_t detail = 0;
    const int64_t cap = P.lay.cap_rows;
    for (int d = 0; d < R; ++d) {
      if (s_slot[d] < 0 || s_slot[d] >= P.num_slots) {
        err = EPB_ERR_CONFIG;
        detail = 0x10000 + d;
      }
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
    if (err) {
      *s_abort = err;
      rv.host->err_detail = detail;
      rv.host->err_code = err;
    }
  }
  if (lane == 0 && *s_abort == 0 && a.num_worst_tokens > 0 && s_rpm[R - 1][me] > a.num_worst_tokens) {
    // more rows than the caller's num_worst_tokens views: the rows still land
    // inside the slot (capacity is checked above) but the caller cannot see
    // them all; reported, not aborted (only this rank's sizing is wrong)
    rv.host->err_detail = ((int64_t)s_rpm[R - 1][me] << 8) | me;
    rv.host->err_code = EPB_ERR_CONFIG;
  }
  __syncwarp();
  const int ab = *s_abort;
  if (lane < R) {
    const int d = lane;
    const int mine = s_rpm[me][d] - (me > 0 ? s_rpm[me - 1][d] : 0);
    int pre = 0;  // send-staging start: my rows to lower peers (the local destination is written in place)
    for (int q = 0; q < d; ++q)
      if (q != me) pre += s_rpm[me][q] - (me > 0 ? s_rpm[me - 1][q] : 0);
    st_relaxed_sys(&sc->plan[0][d], tagged(ab ? kNotifyAbort : (uint32_t)s_slot[d], epoch));
    st_relaxed_sys(&sc->plan[1][d], tagged((uint32_t)(me > 0 ? s_rpm[me - 1][d] : 0), epoch));
    st_relaxed_sys(&sc->plan[2][d], tagged((uint32_t)mine, epoch));
    st_relaxed_sys(&sc->plan[3][d], tagged((uint32_t)pre, epoch));
  }
  if (lane == 0) {
    sc->abort = ab;
    // the host sizes its receive tensors from this word (tagged, HostInfo)
    st_relaxed_sys(&rv.host->notify[0], tagged(ab ? kNotifyAbort : (uint32_t)s_rpm[R - 1][me], P.host_seq[lr]));
  }
  trace_mark(rv, 5);
  for (int i = lane; i < R * R; i += 32) a.rank_prefix_matrix[i] = s_rpm[i / R][i % R];
}

// Proxy transport: WRITE TransferCmds (command.py layout, offsets relative to
// the arena start) for every array of the rows I send to each peer, then one
// ATOMIC (+1 on the peer's ht_sig[0][me]) — sent even for zero rows or an
// aborted call, so the per-source counters stay in step with the calls.
__device__ __noinline__ void push_dispatch_cmds(const DispatchParams& P, int lr, const int32_t* slot,
                                                const int32_t* base, const int32_t* mine, const int32_t* pre,
                                                bool aborted) {
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank;
  const epb_recv_layout_t& Lo = P.lay;
  const int64_t arena = (int64_t)kRegionHeader;
  const int64_t row_bytes = (int64_t)a.hidden * a.elem_bytes;
  const int64_t sizes[5] = {row_bytes, (int64_t)a.num_scales * 4, (a.topk_idx ? (int64_t)a.num_topk * 8 : 0),
                            (a.topk_idx && a.topk_weights ? (int64_t)a.num_topk * 4 : 0), 4};
  const int64_t offs[5] = {Lo.off_x, Lo.off_scales, Lo.off_topk_idx, Lo.off_topk_w, Lo.off_src_idx};
  for (int d = 0; d < R; ++d) {
    if (d == me) continue;
    const int ch = d % P.fifo_channels;
    uint64_t lo, hi;
    if (!aborted && mine[d] > 0) {
      const int64_t src_slot = Lo.send_off - arena;
      const int64_t dst_slot = Lo.slot0_off + (int64_t)slot[d] * Lo.slot_bytes - arena;
      for (int f = 0; f < 5; ++f) {
        if (sizes[f] == 0) continue;
        const int64_t so = src_slot + offs[f] + (int64_t)pre[d] * sizes[f];
        const int64_t dof = dst_slot + offs[f] + (int64_t)base[d] * sizes[f];
        cmd_pack_dev(EPB_CMD_WRITE, d, ch, so, dof, (int64_t)mine[d] * sizes[f], 0, lo, hi);
        if (fifo_push(rv, ch, lo, hi) < 0) return;
      }
    }
    cmd_pack_dev(EPB_CMD_ATOMIC, d, ch, 0, offsetof(Meta, ht_sig) + sizeof(uint64_t) * me, 1, 0, lo, hi);
    if (fifo_push(rv, ch, lo, hi) < 0) return;
  }
}

// Row metadata of token t: lane j < k holds topk_idx / weight j, lanes hold
// up to two of the S scales (S <= 64).
constexpr int kMetaTok = 2;
__device__ __forceinline__ void meta_load(const epb_dispatch_args_t& a, int t, int lane, int64_t& e, float& w,
                                          float* sc) {
  const int k = a.num_topk, S = a.num_scales;
  e = (a.topk_idx != nullptr && lane < k) ? a.topk_idx[(size_t)t * k + lane] : -1;
  w = (a.topk_weights != nullptr && lane < k) ? a.topk_weights[(size_t)t * k + lane] : 0.0f;
  sc[0] = (a.x_scales != nullptr && lane < S) ? a.x_scales[(size_t)t * S + lane] : 0.0f;
  sc[1] = (a.x_scales != nullptr && lane + 32 < S) ? a.x_scales[(size_t)t * S + lane + 32] : 0.0f;
}
__device__ __forceinline__ void meta_store(const DispatchParams& P, int lr, int t, int tt, const int32_t* s_pos,
                                           char* const* s_dst, const int32_t* s_rb, int64_t e, float w,
                                           const float* sc, int lane) {
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = P.rv[lr].world, k = a.num_topk, S = a.num_scales;
  const int L = (a.topk_idx != nullptr && a.num_experts > 0) ? a.num_experts / R : 0;
  for (int d = 0; d < R; ++d) {
    const int p = s_pos[tt * R + d];
    if (p < 0) continue;
    const size_t row = (size_t)(s_rb[d] + p);
    char* slot = s_dst[d];
    if (a.x_scales != nullptr) {
      float* ds = reinterpret_cast<float*>(slot + P.lay.off_scales) + row * S;
      if (lane < S) ds[lane] = sc[0];
      if (lane + 32 < S) ds[lane + 32] = sc[1];
    }
    if (a.topk_idx != nullptr && lane < k) {
      const int64_t le = (e >= (int64_t)d * L && e < (int64_t)(d + 1) * L) ? e - (int64_t)d * L : -1;
      reinterpret_cast<int64_t*>(slot + P.lay.off_topk_idx)[row * k + lane] = le;
      if (a.topk_weights != nullptr)
        reinterpret_cast<float*>(slot + P.lay.off_topk_w)[row * k + lane] = le >= 0 ? w : 0.0f;
    }
    if (lane == 0) reinterpret_cast<int32_t*>(slot + P.lay.off_src_idx)[row] = t;
  }
}

__global__ void __launch_bounds__(kDispatchThreads, 1) dispatch_kernel(const __grid_constant__ DispatchParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, C = gridDim.x, c = blockIdx.x, T = a.num_tokens;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  Scratch* sc = scratch_of(rv.base);
  extern __shared__ int32_t s_pos[];  // [Tc][R] row of the token inside its channel's run to d, or -1
  __shared__ int32_t s_cnt[kMaxRanks][kMaxChannels];  // block 0: every channel's counts
  __shared__ int32_t s_rpm[kMaxRanks][kMaxRanks];     // block 0: counts[src][dst], then prefix over src
  __shared__ int32_t s_slot[kMaxRanks];
  __shared__ char* s_dst[kMaxRanks];
  __shared__ int32_t s_rb[kMaxRanks];
  __shared__ int32_t s_chx[kMaxRanks];
  __shared__ int32_t s_slotv[kMaxRanks], s_base[kMaxRanks], s_mine[kMaxRanks], s_pre[kMaxRanks];
  __shared__ int s_abort;
  __shared__ uint32_t s_epoch, s_target;
  trace_mark(rv, 0);
  if (tid == 0) {
    s_abort = 0;
    norm_call_begin(rv, 0, gridDim.x, &s_epoch, &s_target);
  }
  __syncthreads();
  const uint32_t epoch = s_epoch, target = s_target;
  if (c == 0 && warp >= R && warp < 2 * R) post_expert_counts(P, lr, warp - R, epoch);

  // 1. channel-relative positions and per-(destination, channel) counts
  // channel c = a contiguous token range (solo: channel 0 is empty, the
  // tokens are spread over channels 1..C-1)
  const int Tc = P.solo ? (T + C - 2) / (C - 1) : (T + C - 1) / C;
  const int t0 = P.solo ? (c == 0 ? 0 : (c - 1) * Tc) : c * Tc;
  const int nt = (P.solo && c == 0) ? 0 : max(0, min(T, t0 + Tc) - t0);
  if (warp < R) {
    const int d = warp;
    int run = 0;
    for (int g = 0; g < nt; g += 32) {
      const int tt = g + lane;
      const bool in = tt < nt && a.is_token_in_rank[(size_t)(t0 + tt) * R + d] != 0;
      const unsigned b = __ballot_sync(0xffffffffu, in);
      if (tt < nt) s_pos[tt * R + d] = in ? run + __popc(b & ((1u << lane) - 1)) : -1;
      run += __popc(b);
    }
    if (lane == 0) st_relaxed_sys(&sc->ch_cnt[d][c], tagged((uint32_t)run, epoch));
  }
  __syncthreads();

  // 2. block 0 exchanges counts with the peers and publishes the plan; the
  //    other blocks read their part of it (tagged words, one warp polls)
  if (c == 0) {
    exchange_counts(P, lr, C, s_cnt, s_rpm, s_slot, &s_abort, epoch);
    __syncthreads();
  }
  if (P.perblock && c > 0) {
    // my channel's offset in my run to each d: tokens before t0 that go to d
    __shared__ int s_before[kMaxRanks];
    if (tid < R) s_before[tid] = 0;
    __syncthreads();
    int n[kMaxRanks];
#pragma unroll
    for (int d = 0; d < kMaxRanks; ++d) n[d] = 0;
    // 16-byte loads over the [t0, R] bool bytes (R | 16: byte j of a word is
    // destination j % R): one load round for the whole prefix instead of one
    // dependent byte-load round per 512 tokens
    int t_scalar = 0;
    if (16 % R == 0 && (reinterpret_cast<uintptr_t>(a.is_token_in_rank) & 15) == 0) {
      const int nw16 = (t0 * R) >> 4;
      const uint4* ir4 = reinterpret_cast<const uint4*>(a.is_token_in_rank);
      for (int i = tid; i < nw16; i += blockDim.x) {
        const uint4 w = ir4[i];
        const uint32_t q[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t b = (q[j >> 2] >> (8 * (j & 3))) & 0xffu;
#pragma unroll
          for (int d = 0; d < kMaxRanks; ++d)
            if (d < R && j % R == d) n[d] += b != 0;
        }
      }
      t_scalar = (nw16 << 4) / R;
    }
    for (int t = t_scalar + tid; t < t0; t += blockDim.x) {
      uint64_t bits = 0;  // the token's R bool bytes (one aligned load for R = 2, 4, 8)
      const uint8_t* row = a.is_token_in_rank + (size_t)t * R;
      if (R == 8) bits = *reinterpret_cast<const uint64_t*>(row);
      else if (R == 4) bits = *reinterpret_cast<const uint32_t*>(row);
      else if (R == 2) bits = *reinterpret_cast<const uint16_t*>(row);
      else
        for (int d = 0; d < R; ++d) bits |= (uint64_t)row[d] << (8 * d);
#pragma unroll
      for (int d = 0; d < kMaxRanks; ++d) n[d] += ((bits >> (8 * d)) & 0xff) != 0;
    }
#pragma unroll
    for (int d = 0; d < kMaxRanks; ++d) {
      if (d >= R) break;
      const int v = __reduce_add_sync(0xffffffffu, n[d]);
      if (lane == 0 && v) atomicAdd(&s_before[d], v);
    }
    // warp 0: every source's totals and every destination's slot from my
    // mailbox (the words block 0 of each rank posts), then the same
    // capacity checks block 0 makes (all ranks see the same matrix)
    if (warp == 0) {
      constexpr int kPer = (kMaxRanks * (kMaxRanks + 1) + 31) / 32;
      const Meta* my = meta_of(rv.base);
      const int par = epoch & 1;
      uint64_t v[kPer];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int i = lane + 32 * j, s2 = i / (R + 1), f = i % (R + 1);
        v[j] = i < R * (R + 1) ? ld_relaxed_sys(f < R ? &my->mbox[par][s2].counts_per_rank[f] : &my->mbox[par][s2].slot)
                               : tagged(0, epoch);
      }
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int i = lane + 32 * j, s2 = i / (R + 1), f = i % (R + 1);
        if (i < R * (R + 1)) {
          const uint64_t* w = f < R ? &my->mbox[par][s2].counts_per_rank[f] : &my->mbox[par][s2].slot;
          const uint32_t x = (uint32_t)v[j] == epoch ? (uint32_t)(v[j] >> 32) : wait_tagged(rv, w, epoch, 0x1a0 + s2, 64);
          if (x == kNotifyAbort) s_abort = EPB_ERR_DEADLOCK;
          if (f < R) s_rpm[s2][f] = (int)x;
          else s_slot[s2] = (int)x;
        }
      }
      __syncwarp();
      if (lane < R) {  // inclusive prefix over source rank, column d
        int run = 0;
        for (int s2 = 0; s2 < R; ++s2) {
          run += s_rpm[s2][lane];
          s_rpm[s2][lane] = run;
        }
      }
      __syncwarp();
      if (lane == 0) {
        const int64_t cap = P.lay.cap_rows;
        bool bad = false;
        for (int d = 0; d < R; ++d) bad |= s_slot[d] < 0 || s_slot[d] >= P.num_slots || s_rpm[R - 1][d] > cap;
        for (int s2 = 0; s2 < R; ++s2) {
          int sent = 0;
          for (int d = 0; d < R; ++d) sent += s_rpm[s2][d] - (s2 > 0 ? s_rpm[s2 - 1][d] : 0);
          bad |= sent > cap;
        }
        if (bad) s_abort = EPB_ERR_CONFIG;  // block 0 reports it; this block just does not copy
      }
    }
    __syncthreads();
    if (tid < R) {
      const int d = tid;
      s_slotv[d] = s_slot[d];
      s_base[d] = me > 0 ? s_rpm[me - 1][d] : 0;
      s_chx[d] = s_before[d];
    }
  } else if (P.solo && c > 0) {
    // my channel offset = tokens before t0 that go to rank 0 (read straight
    // from is_token_in_rank: <= T bytes, one load round); slot and base are mine
    __shared__ int s_before;
    if (tid == 0) s_before = 0;
    __syncthreads();
    int n = 0;
    int i_scalar = 0;
    if ((reinterpret_cast<uintptr_t>(a.is_token_in_rank) & 15) == 0) {  // 16 bool bytes per load
      const uint4* ir4 = reinterpret_cast<const uint4*>(a.is_token_in_rank);
      for (int i = tid; i < (t0 >> 4); i += blockDim.x) {
        const uint4 w = ir4[i];
        n += __popc(w.x & 0x01010101u) + __popc(w.y & 0x01010101u) + __popc(w.z & 0x01010101u) +
             __popc(w.w & 0x01010101u);
      }
      i_scalar = t0 & ~15;
    }
    for (int i = i_scalar + tid; i < t0; i += blockDim.x) n += a.is_token_in_rank[i] != 0;
    n = __reduce_add_sync(0xffffffffu, n);
    if (lane == 0 && n) atomicAdd(&s_before, n);
    __syncthreads();
    if (tid == 0) {
      s_slotv[0] = a.recv_slot;
      s_base[0] = 0;
      s_chx[0] = s_before;
    }
  } else if (warp == 0 && !(P.solo && c == 0)) {  // block 0, and every block of the proxy transport
    const int nf = P.proxy ? 5 : 3;  // slot, row base, channel offset (+ my count, staging start)
    for (int i = lane; i < nf * R; i += 32) {
      const int d = i % R, f = i / R;
      const uint64_t* w = f == 2 ? &sc->ch_excl[d][c] : &sc->plan[f < 2 ? f : f - 1][d];
      const uint32_t v = wait_tagged(rv, w, epoch, 0x190, c == 0 ? 0 : 64);
      if (f == 0) {
        if (v == kNotifyAbort) s_abort = EPB_ERR_CONFIG;
        s_slotv[d] = (int)v;
      } else if (f == 1) {
        s_base[d] = (int)v;
      } else if (f == 2) {
        s_chx[d] = (int)v;
      } else if (f == 3) {
        s_mine[d] = (int)v;
      } else {
        s_pre[d] = (int)v;
      }
    }
  }
  __syncthreads();
  if (tid < R && !s_abort) {
    const int d = tid;
    if (P.proxy && d != me) {  // rows for a peer go to my send staging, in the peer's order
      s_dst[d] = rv.base + P.lay.send_off;
      s_rb[d] = s_pre[d] + s_chx[d];
    } else {
      s_dst[d] = rv.peer[d] + P.lay.slot0_off + (int64_t)s_slotv[d] * P.lay.slot_bytes;
      s_rb[d] = s_base[d] + s_chx[d];  // first row of this channel's run at d
    }
  }
  __syncthreads();
  trace_mark(rv, 7);
  trace_mark_max(rv, 11);

  // 3. push rows (block 0's first warps publish the counts meanwhile)
  const int first_copy_warp = c == 0 ? kPublishWarps : 0;
  if (warp < first_copy_warp) publish_counts(P, lr, C, s_abort != 0, epoch);
  if (!s_abort) {
    for (int i = tid; i < nt * R; i += blockDim.x) {  // handle: row of t inside my block at d, or -1
      const int p = s_pos[i];
      a.send_head[(size_t)t0 * R + i] = p < 0 ? -1 : p + s_chx[i % R];
    }
    const size_t row_bytes = (size_t)a.hidden * a.elem_bytes;
    const int n16 = (int)(row_bytes >> 4);
    // Rows move in units of (token, 3.5 KB segment), two units in flight per
    // warp (14 x 16 B loads per lane): the channel's ~28 tokens x 4 segments
    // spread evenly over the block's warps (whole rows left the slowest warp
    // with 2 rows against a mean of 1.75), and each row is read from HBM once
    // and stored to every destination that needs it.
    const int wc = warp - first_copy_warp, nwc = nwarps - first_copy_warp;
    // this warp's first kMetaTok tokens: metadata loads issued now, stored after the rows
    int64_t m_e[kMetaTok];
    float m_w[kMetaTok], m_sc[kMetaTok][2];
#pragma unroll
    for (int q = 0; q < kMetaTok; ++q) {
      const int tt = wc + q * nwc;
      m_e[q] = -1;
      m_w[q] = 0.0f;
      m_sc[q][0] = m_sc[q][1] = 0.0f;
      if (!P.notify_only && wc >= 0 && tt < nt) meta_load(a, t0 + tt, lane, m_e[q], m_w[q], m_sc[q]);
    }
    if (P.tma && !P.notify_only) {
      // Bulk-copy path: warp w < kTmaWarps (of the copy warps), lane 0, runs a
      // kTmaStages-deep ring: unit i = (token, segment) is bulk-loaded into its
      // stage (mbarrier), bulk-stored to every destination (one bulk group),
      // and its stage is refilled with unit i + kTmaStages - 1 once the group of
      // unit i - 1 has finished reading shared memory.
      __shared__ __align__(8) uint64_t s_bar[kTmaWarps][kTmaStages];
      extern __shared__ __align__(128) uint8_t s_dyn[];
      const int seg = P.tma_seg, nseg = (int)((row_bytes + seg - 1) / seg);
      const int tma_units = nt * nseg;
      if (wc >= 0 && wc < kTmaWarps && lane == 0) {
        uint8_t* ring = s_dyn + P.tma_smem_off + (size_t)wc * kTmaStages * seg;
        const uint64_t pol = l2_policy_evict_last();
        uint64_t* bar = s_bar[wc];
        for (int st = 0; st < kTmaStages; ++st) mbar_init(&bar[st], 1);
        fence_async_shared();
        const int n_my = tma_units > wc ? (tma_units - wc + kTmaWarps - 1) / kTmaWarps : 0;
        auto unit_src = [&](int i, uint32_t& len) -> const char* {
          const int u = wc + i * kTmaWarps, tt = u / nseg, sg = u % nseg;
          const size_t off = (size_t)sg * seg;
          len = (uint32_t)min((size_t)seg, row_bytes - off);
          return static_cast<const char*>(a.x) + (size_t)(t0 + tt) * row_bytes + off;
        };
        auto issue_load = [&](int i) {
          uint32_t len;
          const char* src = unit_src(i, len);
          const int st = i % kTmaStages;
          mbar_expect_tx(&bar[st], len);
          bulk_load(ring + (size_t)st * seg, src, len, &bar[st]);
        };
        for (int i = 0; i < min(n_my, kTmaStages - 1); ++i) issue_load(i);
        for (int i = 0; i < n_my; ++i) {
          const int st = i % kTmaStages;
          while (!mbar_try_wait(&bar[st], (uint32_t)((i / kTmaStages) & 1))) {
          }
          const int u = wc + i * kTmaWarps, tt = u / nseg, sg = u % nseg;
          const size_t off = (size_t)sg * seg;
          const uint32_t len = (uint32_t)min((size_t)seg, row_bytes - off);
          for (int d = 0; d < R; ++d) {
            const int p = s_pos[tt * R + d];
            if (p < 0) continue;
            char* dst = s_dst[d] + P.lay.off_x + (size_t)(s_rb[d] + p) * row_bytes + off;
            if (P.tma == 2) bulk_store_hint(dst, ring + (size_t)st * seg, len, pol);
            else bulk_store(dst, ring + (size_t)st * seg, len);
          }
          bulk_commit();
          if (i + kTmaStages - 1 < n_my) {
            bulk_wait_read<1>();  // unit i - 1's stores have read the stage unit i + S - 1 reuses
            issue_load(i + kTmaStages - 1);
          }
        }
        bulk_wait_all();
      }
    }
    constexpr int kSeg = 32 * kCopyUnroll;
    const int segs = (n16 + kSeg - 1) / kSeg;
    const int units = (P.notify_only || P.tma) ? 0 : nt * segs;
    for (int u = wc; wc >= 0 && u < units; u += 2 * nwc) {
      int4 v[2][kCopyUnroll];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int uu = u + q * nwc;
        if (uu >= units) break;
        const int tt = uu / segs, i0 = (uu % segs) * kSeg;
        const int4* src = reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + (size_t)(t0 + tt) * row_bytes);
#pragma unroll
        for (int j = 0; j < kCopyUnroll; ++j) {
          const int i = i0 + j * 32 + lane;
          if (i < n16) v[q][j] = ld_nc_v4(src + i);
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int uu = u + q * nwc;
        if (uu >= units) break;
        const int tt = uu / segs, i0 = (uu % segs) * kSeg;
        for (int d = 0; d < R; ++d) {
          const int p = s_pos[tt * R + d];
          if (p < 0) continue;
          int4* dst = reinterpret_cast<int4*>(s_dst[d] + P.lay.off_x + (size_t)(s_rb[d] + p) * row_bytes);
#pragma unroll
          for (int j = 0; j < kCopyUnroll; ++j) {
            const int i = i0 + j * 32 + lane;
            if (i < n16) st_v4(dst + i, v[q][j]);
          }
        }
      }
    }
    // per-row metadata: scales, mapped top-k, source index.  The values were
    // loaded before the copy loop (meta_load), so their latency is hidden.
    for (int q = 0; q < kMetaTok; ++q) {
      const int tt = wc + q * nwc;
      if (P.notify_only || wc < 0 || tt >= nt) break;
      meta_store(P, lr, t0 + tt, tt, s_pos, s_dst, s_rb, m_e[q], m_w[q], m_sc[q], lane);
    }
    for (int tt = wc + kMetaTok * nwc; !P.notify_only && wc >= 0 && tt < nt; tt += nwc) {
      int64_t e;
      float w;
      float sc[2];
      meta_load(a, t0 + tt, lane, e, w, sc);
      meta_store(P, lr, t0 + tt, tt, s_pos, s_dst, s_rb, e, w, sc, lane);
    }
  }

  // 4. completion: bar.sync orders every thread's row stores before the
  //    release-add (PTX release cumulativity); block 0 holds the kernel open
  //    until every source's blocks have landed here
  __syncthreads();
  trace_mark(rv, 9);
  trace_mark_max(rv, 12);
  if (P.notify_only) {
    // no rows moved: nothing to signal (the handle outputs are complete when
    // the kernel ends; the ring kernel runs next on the stream)
  } else if (!P.proxy) {
    if (tid < R) {  // the local destination only needs gpu scope
      if (tid == me) red_release_gpu_add(&meta_of(rv.peer[tid])->disp_done[me], 1u);
      else red_release_sys_add(&meta_of(rv.peer[tid])->disp_done[me], 1u);
    }
    if (c == 0 && a.num_worst_tokens > 0 && a.topk_idx != nullptr && !s_abort) {
      // num_worst_tokens: receive rows past the real count carry no expert
      // (DeepEP semantics); block 0 marks them while the peers' rows land
      const int64_t n_real = (int64_t)s_rpm[R - 1][me] * a.num_topk;
      const int64_t n_all = (int64_t)a.num_worst_tokens * a.num_topk;
      int64_t* ti = reinterpret_cast<int64_t*>(rv.base + P.lay.slot0_off + (int64_t)a.recv_slot * P.lay.slot_bytes +
                                               P.lay.off_topk_idx);
      for (int64_t i = n_real + tid; i < n_all; i += blockDim.x) ti[i] = -1;
    }
    if (c == 0 && tid < R) wait_geq(rv, &meta_of(rv.base)->disp_done[tid], target, 0x200 + tid);
  } else {
    // proxy transport: the last of my blocks to finish hands the peers' rows
    // to the CPU proxy — one WRITE per array and destination (contiguous in
    // my staging and in the peer's slot), then an ATOMIC on the peer's
    // ht_sig[0][me]; FIFO order on the channel puts the data first
    if (tid == 0) {
      const uint32_t old = atom_add_acq_rel_gpu(&meta_of(rv.base)->disp_done[me], 1u);
      if (old + 1 == target) push_dispatch_cmds(P, lr, s_slotv, s_base, s_mine, s_pre, s_abort != 0);
    }
    // the peers' rows are awaited by dispatch_proxy_wait_kernel, launched next
    // on the stream: no block of this kernel stays resident spinning on copies
    // the proxy issues (a copy-engine transfer was observed to stall behind one)
  }
  trace_mark(rv, 10);
  if (tid == 0) norm_call_end(rv, 0, epoch, target);
}

// Proxy transport: one block per local rank waits until every peer's rows
// (and its ATOMIC) have landed; my own rows were written by the kernel above.
__global__ void dispatch_proxy_wait_kernel(const __grid_constant__ DispatchParams P) {
  const RankView& rv = P.rv[blockIdx.x];
  const int tid = threadIdx.x;
  if (tid < rv.world && tid != rv.rank)
    wait_geq64(rv, &meta_of(rv.base)->ht_sig[0][tid], P.ht_calls[blockIdx.x], 0x220 + tid, 500);
}

}  // namespace epb

using namespace epb;

static int dispatch_launch(epb_t* const* ctxs, int n_local, const epb_dispatch_args_t* args, int num_channels,
                           void* stream, int notify_only) {
  if (int e = check_group(ctxs, n_local)) return e;
  if (num_channels <= 0 || num_channels > kMaxChannels)
    return epb_set_error(EPB_ERR_CONFIG, "num_channels out of range");
  DispatchParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_local = n_local;
  P.num_slots = std::max(1, ctxs[0]->cfg.num_recv_slots);
  P.proxy = ctxs[0]->cfg.ht_transport == EPB_HT_PROXY ? 1 : 0;
  P.notify_only = notify_only;
  P.fifo_channels = ctxs[0]->cfg.fifo_channels;
  for (int i = 0; i < n_local; ++i) {
    if (ctxs[i]->cfg.ht_transport != ctxs[0]->cfg.ht_transport)
      return epb_set_error(EPB_ERR_CONFIG, "all ranks of a group must use the same ht_transport");
    if (P.proxy && (ctxs[i]->cfg.fifo_channels <= 0 || !ctxs[i]->proxy))
      return epb_set_error(EPB_ERR_CONFIG, "ht_transport=proxy needs FIFO channels and a running proxy");
  }
  int max_tc = 1;
  for (int i = 0; i < n_local; ++i) {
    const epb_dispatch_args_t& a = args[i];
    if (a.elem_bytes != 1 && a.elem_bytes != 2) return epb_set_error(EPB_ERR_CONFIG, "elem_bytes must be 1 or 2");
    if (((size_t)a.hidden * a.elem_bytes) % 16 != 0) return epb_set_error(EPB_ERR_CONFIG, "row bytes must be 16-aligned");
    if (a.num_scales > 64) return epb_set_error(EPB_ERR_CONFIG, "at most 64 scales per row (hidden <= 8192 with FP8)");
    if (a.num_topk > 32) return epb_set_error(EPB_ERR_CONFIG, "num_topk must be <= 32");
    if (a.num_experts > 0 &&
        (a.num_experts % ctxs[i]->world != 0 || a.num_experts / ctxs[i]->world > kMaxLocalExperts))
      return epb_set_error(EPB_ERR_CONFIG, "num_experts must be a multiple of world (<= 1024 local experts)");
    if (!notify_only)
      if (int e = compute_recv_layout(ctxs[i], a.hidden, a.num_topk, &P.lay)) return e;
    max_tc = std::max(max_tc, (a.num_tokens + num_channels - 1) / num_channels);
    if (ctxs[0]->world > 1 && !P.proxy && !notify_only && !std::getenv("EPB_PLAN_HOP")) P.perblock = 1;
    if (n_local == 1 && ctxs[0]->world == 1 && !P.proxy && !notify_only && num_channels >= 2 &&
        (int64_t)a.num_tokens <= P.lay.cap_rows) {
      P.solo = 1;
      max_tc = std::max(max_tc, (a.num_tokens + num_channels - 2) / (num_channels - 1));
    }
  }
  size_t smem = sizeof(int32_t) * (size_t)max_tc * ctxs[0]->world;
  if (smem > 160 * 1024) return epb_set_error(EPB_ERR_CONFIG, "too many tokens per channel; raise num_sms");
  // Bulk-copy rows (TMA engine) when the dispatch runs on a small SM budget:
  // at 20 / 24 / 48 channels it moves the DS-V3 rows 11-13 % faster than the
  // warp copy; on the whole GPU the warp copy wins the step (the combine behind
  // a bulk-copied dispatch ran slower: 59 against 52 us per N=1 step,
  // profiles/r02_summary.md).  EPB_TMA=0 / 1 / 2 forces off / on / on with an
  // L2 evict_last hint on the bulk stores.
  static const int tma_env = [] {
    const char* v = std::getenv("EPB_TMA");
    return v ? std::atoi(v) : -1;
  }();
  const int tma_want = tma_env >= 0 ? tma_env : (num_channels <= kTmaAutoChannels ? 1 : 0);
  P.tma = 0;
  if (tma_want && !notify_only) {
    const size_t rb = (size_t)args[0].hidden * args[0].elem_bytes;
    const int nseg = (int)((rb + kTmaSegMax - 1) / kTmaSegMax);
    const int seg = (int)align_up((rb + nseg - 1) / nseg, 16);
    const size_t off = align_up(smem, 128);
    const size_t need = off + (size_t)kTmaWarps * kTmaStages * seg;
    bool ok = need <= 200 * 1024;
    for (int i = 0; i < n_local && ok; ++i)
      ok = (reinterpret_cast<uintptr_t>(args[i].x) & 15) == 0 && (size_t)args[i].hidden * args[i].elem_bytes == rb;
    if (ok) {
      P.tma = tma_want;  // 2: bulk stores carry an L2 evict_last hint
      P.tma_seg = seg;
      P.tma_smem_off = (int)off;
      smem = need;
    }
  }
  // max shared carveout: the N=1 step (layout, dispatch, combine back to back)
  // took 70 us with the driver's choice and 63 us with this, although the
  // dispatch alone is ~2 us slower; the gain is in the gap after the dispatch
  // (profiles/r01d_summary.md).  The combine keeps the driver's choice.
  epb_set_carveout((const void*)dispatch_kernel, !epb_carveout_skip("dispatch"));
  EPB_CUDA(epb_ensure_smem((const void*)dispatch_kernel, smem));
  const int max_active = epb_max_active_blocks((const void*)dispatch_kernel, kDispatchThreads, smem);
  if ((int64_t)num_channels * n_local > (int64_t)max_active * ctxs[0]->num_sms)
    return epb_set_error(EPB_ERR_CONFIG, "num_channels x ranks exceeds the co-resident grid; lower num_sms");
  for (int i = 0; i < n_local; ++i) {
    epb_ctx* c = ctxs[i];
    P.host_seq[i] = ++c->host_seq;
    if (P.proxy) P.ht_calls[i] = ++c->ht_disp_calls;
    P.rv[i] = c->view();
    P.a[i] = args[i];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(epb_launch_grid_sync((void*)dispatch_kernel, dim3(num_channels, n_local), dim3(kDispatchThreads),
                                       kargs, smem, st));
  if (P.proxy) {
    dispatch_proxy_wait_kernel<<<n_local, 32, 0, st>>>(P);
    EPB_CUDA(cudaGetLastError());
    // no host sync: the stall that once held the proxy's copies behind work
    // enqueued after this wait was the lazy load of the next kernel (fixed by
    // epb_create's kernel preload); EPB_PROXY_SYNC=1 restores the sync
    if (std::getenv("EPB_PROXY_SYNC")) EPB_CUDA(cudaStreamSynchronize(st));
  }
  return EPB_OK;
}

extern "C" int epb_dispatch(epb_t* const* ctxs, int n_local, const epb_dispatch_args_t* args, int num_channels,
                            void* stream) {
  if (ctxs && n_local > 0 && ctxs[0] && ctxs[0]->cfg.ht_transport == EPB_HT_RING)
    return epb_set_error(EPB_ERR_CONFIG, "ht_transport=ring: use epb_dispatch_notify + epb_ring_dispatch");
  return dispatch_launch(ctxs, n_local, args, num_channels, stream, 0);
}

extern "C" int epb_dispatch_notify(epb_t* const* ctxs, int n_local, const epb_dispatch_args_t* args,
                                   int num_channels, void* stream) {
  return dispatch_launch(ctxs, n_local, args, num_channels, stream, 1);
}

extern "C" int epb_wait_notify(epb_t* ctx, int64_t* num_recv, int32_t* num_recv_per_expert, int num_local_experts,
                               double timeout_s) {
  if (!ctx) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
  if (num_recv_per_expert && (num_local_experts < 0 || num_local_experts > kMaxLocalExperts))
    return epb_set_error(EPB_ERR_PROTOCOL, "num_local_experts out of range");
  const uint32_t want = ctx->host_seq;
  const int nwords = 1 + (num_recv_per_expert ? num_local_experts : 0);
  volatile uint64_t* w = ctx->host->notify;
  auto t0 = std::chrono::steady_clock::now();
  int i = 0;
  uint64_t v = 0;
  while (i < nwords) {
    v = w[i];
    if ((uint32_t)v == want) {
      if (i == 0) {
        if ((uint32_t)(v >> 32) == kNotifyAbort) break;
        if (num_recv) *num_recv = (int64_t)(v >> 32);
      } else {
        num_recv_per_expert[i - 1] = (int32_t)(v >> 32);
      }
      ++i;
      continue;
    }
    if (ctx->host->err_code != 0) break;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
      cudaError_t ce = cudaGetLastError();
      if (ce != cudaSuccess) return epb_cuda_check(ce, "dispatch kernel");
      return epb_set_error(EPB_ERR_DEADLOCK, "dispatch timed out waiting for the peers' counts");
    }
  }
  if (i < nwords) {  // aborted: the error word is written (system scope) before the kernel returns
    while (ctx->host->err_code == 0 &&
           std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() <= timeout_s) {
    }
    char buf[160];
    snprintf(buf, sizeof(buf), "device reported error %lld (detail 0x%llx) in dispatch",
             (long long)ctx->host->err_code, (long long)ctx->host->err_detail);
    const int code = ctx->host->err_code != 0 ? (int)ctx->host->err_code : EPB_ERR_DEADLOCK;
    return epb_set_error(code, buf);
  }
  return EPB_OK;
}

// Load this file's kernels now (see epb_preload_kernels, api.cpp).
cudaError_t epb_preload_dispatch() {
  cudaFuncAttributes attr;
  for (const void* fn : {(const void*)dispatch_kernel, (const void*)dispatch_proxy_wait_kernel})
    if (cudaError_t e = cudaFuncGetAttributes(&attr, fn)) return e;
  return cudaSuccess;
}
