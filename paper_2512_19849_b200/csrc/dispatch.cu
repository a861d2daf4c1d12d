// dispatch.cu — normal-mode (high-throughput) dispatch on sm_100a, one
// cooperative kernel per call:
//
//   1. every block = one channel (a contiguous token range); warp d ballots
//      the channel's tokens for destination d -> positions + per-channel count
//   2. grid barrier; block 0 runs the count exchange ("notify"): channel
//      prefix sums, one mailbox message per peer over NVLink (per-rank totals,
//      per-channel counts, per-expert counts, my receive slot), waits for every
//      peer's message, derives the rank prefix matrix and this rank's plan
//      (destination slot address + first row per destination), publishes the
//      plan with a gpu-scope release, then publishes the receive counts to the
//      host (pinned memory) for the caller's tensor shapes
//   3. all blocks read the plan and push every deduplicated row straight into
//      its final row of the destination's receive slot: one HBM read per row,
//      one 16-byte store per lane per destination (NVLink for peers)
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
#include <cstring>

#include "common.cuh"
#include "ctx.h"

namespace epb {

constexpr int kDispatchThreads = 512;
constexpr int kCopyUnroll = 7;  // 7 x 16 B per lane in flight = 3.5 KB per warp

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
  uint32_t epoch[kMaxLocal];   // per-call epoch: mailbox parity and the go flag value
  uint32_t target[kMaxLocal];  // cumulative arrive / done target (sum of grid widths so far)
  RankView rv[kMaxLocal];
  epb_dispatch_args_t a[kMaxLocal];
  epb_recv_layout_t lay;
};

// Block 0's part: the cross-rank count exchange and the plan.
__device__ __noinline__ void exchange_counts(const DispatchParams& P, int lr, int C) {
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, T = a.num_tokens;
  const uint32_t epoch = P.epoch[lr];
  const int par = epoch & 1;
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  Scratch* sc = scratch_of(rv.base);
  Meta* my = meta_of(rv.base);
  __shared__ int32_t s_cnt[kMaxRanks][kMaxChannels];
  __shared__ int32_t s_tot[kMaxRanks];
  __shared__ int32_t s_rpm[kMaxRanks][kMaxRanks];

  __shared__ int32_t s_exp[kMaxRanks * kMaxLocalExperts];  // num_tokens_per_expert, prefetched
  const int E = a.num_tokens_per_expert != nullptr ? a.num_experts : 0;
  for (int e = tid; e < E; e += nthr) s_exp[e] = __ldg(&a.num_tokens_per_expert[e]);  // overlaps the barrier
  if (tid == 0) wait_geq_gpu(rv, &sc->disp_arrive, P.target[lr], 0x180);
  __syncthreads();
  for (int i = tid; i < R * C; i += nthr) s_cnt[i / C][i % C] = __ldcg(&sc->ch_cnt[i / C][i % C]);
  __syncthreads();
  trace_mark(rv, 1);
  if (warp < R) {
    const int tot = warp_scan_row(&s_cnt[warp][0], a.channel_prefix_matrix + warp * C, &sc->ch_excl[warp][0], C, lane);
    if (lane == 0) s_tot[warp] = tot;
  }
  __syncthreads();
  trace_mark(rv, 2);

  // post my counts into every peer's mailbox (warp d -> peer d), then stamp the epoch
  const int L = a.num_experts > 0 ? a.num_experts / R : 0;
  if (warp < R) {
    const int d = warp;
    NotifyMsg* msg = &meta_of(rv.peer[d])->mbox[par][me];
    for (int i = lane; i < R; i += 32) msg->counts_per_rank[i] = s_tot[i];
    if (lane == 0) {
      msg->slot = a.recv_slot;
      msg->num_tokens = T;
    }
    for (int i = lane; i < C; i += 32) msg->channel_counts[i] = s_cnt[d][i];
    if (a.num_tokens_per_expert != nullptr)
      for (int e = lane; e < L; e += 32) msg->expert_counts[e] = s_exp[d * L + e];
    __syncwarp();
    if (lane == 0) st_release_sys(&meta_of(rv.peer[d])->mbox_flag[par][me], epoch);
  }
  trace_mark(rv, 3);
  if (tid < R) wait_geq(rv, &my->mbox_flag[par][tid], epoch, 0x100 + tid);
  __syncthreads();
  trace_mark(rv, 4);

  // the rank prefix matrix first (all the plan needs); the per-channel receive
  // prefix is a handle output and is computed after the plan is published
  if (tid < R * R) s_rpm[tid / R][tid % R] = __ldcg(&my->mbox[par][tid / R].counts_per_rank[tid % R]);
  __syncthreads();
  if (warp == 0 && lane < R) {
    const int d = lane;  // inclusive prefix over source rank, column d
    int run = 0;
    for (int s = 0; s < R; ++s) {
      run += s_rpm[s][d];
      s_rpm[s][d] = run;
      a.rank_prefix_matrix[s * R + d] = run;
    }
  }
  __syncthreads();

  // plan + capacity checks (every rank sees the same matrix, so all abort together)
  if (tid < R) {
    const int d = tid;
    const int slot_d = __ldcg(&my->mbox[par][d].slot);
    sc->dst_rows[d] = reinterpret_cast<uint64_t>(rv.peer[d] + P.lay.slot0_off + (int64_t)slot_d * P.lay.slot_bytes);
    sc->row_base[d] = me > 0 ? s_rpm[me - 1][d] : 0;
  }
  if (tid == 0) {
    int err = 0;
    int64_t detail = 0;
    const int64_t cap = P.lay.cap_rows;
    for (int d = 0; d < R; ++d) {
      const int slot_d = __ldcg(&my->mbox[par][d].slot);
      if (slot_d < 0 || slot_d >= P.num_slots) {
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
    sc->abort = err;
    if (err) {
      rv.host->err_detail = detail;
      rv.host->err_code = err;
    }
  }
  __syncthreads();
  if (tid == 0) st_release_gpu(&sc->disp_go, epoch);  // the plan is visible to the other blocks
  trace_mark(rv, 5);
}

// Block 0, warps [0, kPublishWarps): handle outputs and host publication,
// while block 0's other warps already copy rows.
constexpr int kPublishWarps = 2;
__device__ __noinline__ void publish_counts(const DispatchParams& P, int lr, int C) {
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank;
  const uint32_t epoch = P.epoch[lr];
  const int par = epoch & 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int nthr = kPublishWarps * 32;
  Meta* my = meta_of(rv.base);
  // every source's per-channel counts -> receive channel prefix (handle output)
  for (int d = warp; d < R; d += kPublishWarps)
    warp_scan_row(&my->mbox[par][d].channel_counts[0], a.recv_channel_prefix_matrix + d * C, nullptr, C, lane);
  // receive counts for the caller's tensor shapes
  const int L = a.num_experts > 0 ? a.num_experts / R : 0;
  if (a.num_tokens_per_expert != nullptr) {
    const int align = max(1, a.expert_alignment);
    for (int le = tid; le < L; le += nthr) {
      int n = 0;
      for (int s = 0; s < R; ++s) n += __ldcg(&my->mbox[par][s].expert_counts[le]);
      rv.host->recv_per_expert[le] = (n + align - 1) / align * align;
    }
  }
  if (tid == 0) rv.host->num_recv = a.rank_prefix_matrix[(R - 1) * R + me];
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  if (tid == 0) st_release_sys(const_cast<int64_t*>(&rv.host->notify_epoch), (int64_t)epoch);
  trace_mark(rv, 6);
}

__global__ void __launch_bounds__(kDispatchThreads, 1) dispatch_kernel(const __grid_constant__ DispatchParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_dispatch_args_t& a = P.a[lr];
  const int R = rv.world, me = rv.rank, C = gridDim.x, c = blockIdx.x, T = a.num_tokens;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  Scratch* sc = scratch_of(rv.base);
  extern __shared__ int32_t s_pos[];  // [Tc][R] row of the token inside its channel's run to d, or -1
  __shared__ char* s_dst[kMaxRanks];
  __shared__ int32_t s_rb[kMaxRanks];
  __shared__ int32_t s_chx[kMaxRanks];
  __shared__ int s_abort;
  trace_mark(rv, 0);

  // 1. channel-relative positions and per-(destination, channel) counts
  const int Tc = (T + C - 1) / C;
  const int t0 = c * Tc, nt = max(0, min(T, t0 + Tc) - t0);
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
    if (lane == 0) sc->ch_cnt[d][c] = run;
  }
  __syncthreads();
  if (tid == 0) red_release_gpu_add(&sc->disp_arrive, 1u);

  // 2. block 0 exchanges counts with the peers and publishes the plan
  if (c == 0) {
    exchange_counts(P, lr, C);
  } else {
    if (tid == 0) wait_geq_gpu(rv, &sc->disp_go, P.epoch[lr], 0x190);
    __syncthreads();
  }
  if (tid < R) {
    s_dst[tid] = reinterpret_cast<char*>(__ldcg(reinterpret_cast<const unsigned long long*>(&sc->dst_rows[tid])));
    s_chx[tid] = __ldcg(&sc->ch_excl[tid][c]);          // this channel's offset inside my block at tid
    s_rb[tid] = __ldcg(&sc->row_base[tid]) + s_chx[tid];  // first row of this channel's run at tid
  }
  if (tid == 0) s_abort = __ldcg(&sc->abort);
  __syncthreads();
  trace_mark(rv, 7);

  // 3. push rows (block 0's first warps publish the counts meanwhile)
  const int first_copy_warp = c == 0 ? kPublishWarps : 0;
  if (warp < first_copy_warp) publish_counts(P, lr, C);
  if (!s_abort) {
    for (int i = tid; i < nt * R; i += blockDim.x) {  // handle: row of t inside my block at d, or -1
      const int p = s_pos[i];
      a.send_head[(size_t)t0 * R + i] = p < 0 ? -1 : p + s_chx[i % R];
    }
    const size_t row_bytes = (size_t)a.hidden * a.elem_bytes;
    const int n16 = (int)(row_bytes >> 4);
    const int k = a.num_topk, S = a.num_scales;
    const int L = (a.topk_idx != nullptr && a.num_experts > 0) ? a.num_experts / R : 0;
    for (int tt = warp - first_copy_warp; tt >= 0 && tt < nt; tt += nwarps - first_copy_warp) {
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

  // 4. completion: bar.sync orders every thread's row stores before the
  //    release-add (PTX release cumulativity); block 0 holds the kernel open
  //    until every source's blocks have landed here
  __syncthreads();
  trace_mark(rv, 9);
  if (tid < R) red_release_sys_add(&meta_of(rv.peer[tid])->disp_done[me], 1u);
  if (c == 0 && tid < R) wait_geq(rv, &meta_of(rv.base)->disp_done[tid], P.target[lr], 0x200 + tid);
  trace_mark(rv, 10);
}

}  // namespace epb

using namespace epb;

extern "C" int epb_dispatch(epb_t* const* ctxs, int n_local, const epb_dispatch_args_t* args, int num_channels,
                            void* stream) {
  if (int e = check_group(ctxs, n_local)) return e;
  if (num_channels <= 0 || num_channels > kMaxChannels)
    return epb_set_error(EPB_ERR_CONFIG, "num_channels out of range");
  DispatchParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_local = n_local;
  P.num_slots = std::max(1, ctxs[0]->cfg.num_recv_slots);
  int max_tc = 1;
  for (int i = 0; i < n_local; ++i) {
    const epb_dispatch_args_t& a = args[i];
    if (a.elem_bytes != 1 && a.elem_bytes != 2) return epb_set_error(EPB_ERR_CONFIG, "elem_bytes must be 1 or 2");
    if (((size_t)a.hidden * a.elem_bytes) % 16 != 0) return epb_set_error(EPB_ERR_CONFIG, "row bytes must be 16-aligned");
    if (a.num_experts > 0 &&
        (a.num_experts % ctxs[i]->world != 0 || a.num_experts / ctxs[i]->world > kMaxLocalExperts))
      return epb_set_error(EPB_ERR_CONFIG, "num_experts must be a multiple of world (<= 1024 local experts)");
    if (int e = compute_recv_layout(ctxs[i], a.hidden, a.num_topk, &P.lay)) return e;
    max_tc = std::max(max_tc, (a.num_tokens + num_channels - 1) / num_channels);
  }
  const size_t smem = sizeof(int32_t) * (size_t)max_tc * ctxs[0]->world;
  if (smem > 160 * 1024) return epb_set_error(EPB_ERR_CONFIG, "too many tokens per channel; raise num_sms");
  EPB_CUDA(epb_ensure_smem((const void*)dispatch_kernel, smem));
  const int max_active = epb_max_active_blocks((const void*)dispatch_kernel, kDispatchThreads, smem);
  if ((int64_t)num_channels * n_local > (int64_t)max_active * ctxs[0]->num_sms)
    return epb_set_error(EPB_ERR_CONFIG, "num_channels x ranks exceeds the co-resident grid; lower num_sms");
  for (int i = 0; i < n_local; ++i) {
    epb_ctx* c = ctxs[i];
    P.epoch[i] = ++c->disp_epoch;
    c->disp_cum += (uint32_t)num_channels;
    P.target[i] = c->disp_cum;
    P.rv[i] = c->view();
    P.a[i] = args[i];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(epb_launch_grid_sync((void*)dispatch_kernel, dim3(num_channels, n_local), dim3(kDispatchThreads),
                                       kargs, smem, st));
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
    if (ctx->host->err_code != 0) break;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
      cudaError_t ce = cudaGetLastError();
      if (ce != cudaSuccess) return epb_cuda_check(ce, "dispatch kernel");
      return epb_set_error(EPB_ERR_DEADLOCK, "dispatch timed out waiting for the peers' counts");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  if (ctx->host->err_code != 0) {
    char buf[160];
    snprintf(buf, sizeof(buf), "device reported error %lld (detail 0x%llx) in dispatch",
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
