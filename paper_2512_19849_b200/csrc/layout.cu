// layout.cu — the dispatch layout kernel (DeepEP get_dispatch_layout) and
// the host-side geometry of the normal-mode receive arena.
//
// Layout = the reference's plan_dedup: a
// token goes once to every distinct destination rank among its top-k
// experts (on one NVLink node "node" == rank).
//
// Primary kernel: ONE thread-block cluster of 16 blocks (B200's largest,
// opt-in non-portable size).  Every block stages its slice of the [tokens x k]
// top-k matrix with 16-byte loads, writes is_token_in_rank and builds its
// (expert, rank) histogram in shared memory; after a cluster barrier each
// block sums one slice of the histogram across all 16 blocks through
// distributed shared memory and stores the counts: no zeroing pass, no global
// atomics, no grid barrier.
//
// Fallback (if the cluster launch is refused): one cooperative kernel; block
// 0 zeroes the count outputs while every block histograms its tile, a grid
// barrier orders the zeroing before the blocks' global atomics.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "ctx.h"

namespace epb {

constexpr int kLayoutThreads = 512;  // upper bound for EPB_LAYOUT_THREADS

__global__ void __launch_bounds__(kLayoutThreads) layout_kernel(const int64_t* __restrict__ topk_idx, int T, int k,
                                                                 int E, int R, int32_t* __restrict__ per_rank,
                                                                 int32_t* __restrict__ per_expert,
                                                                 uint8_t* __restrict__ in_rank) {
  extern __shared__ int64_t s_dyn[];
  int64_t* s_topk = s_dyn;                                                        // [blockDim * k]
  int32_t* s_hist = reinterpret_cast<int32_t*>(s_topk + (size_t)blockDim.x * k);  // [E + R]
  const int tid = threadIdx.x, lane = tid & 31;
  if (blockIdx.x == 0) {
    for (int i = tid; i < E; i += blockDim.x) per_expert[i] = 0;
    for (int i = tid; i < R; i += blockDim.x) per_rank[i] = 0;
  }
  for (int i = tid; i < E + R; i += blockDim.x) s_hist[i] = 0;
  const int L = E / R;
  for (int t_first = blockIdx.x * blockDim.x; t_first < T; t_first += gridDim.x * blockDim.x) {
    // stage this tile with coalesced 16-byte loads
    const int n_tok = min((int)blockDim.x, T - t_first);
    const int n_words = n_tok * k;
    const int64_t* src = topk_idx + (size_t)t_first * k;
    __syncthreads();
    if (((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (n_words % 2 == 0)) {
      for (int i = tid; i < n_words / 2; i += blockDim.x)
        reinterpret_cast<int4*>(s_topk)[i] = __ldg(reinterpret_cast<const int4*>(src) + i);
    } else {
      for (int i = tid; i < n_words; i += blockDim.x) s_topk[i] = __ldg(src + i);
    }
    __syncthreads();
    const int t = t_first + tid;
    const bool valid = t < T;
    uint32_t mask = 0;
    for (int j = 0; j < k; ++j) {
      const int64_t e64 = valid ? s_topk[tid * k + j] : -1;
      const int e = (e64 >= 0 && e64 < E) ? (int)e64 : -1;  // out-of-range experts are treated as masked
      if (e >= 0) {
        mask |= 1u << (e / L);  // 32-bit division (the 64-bit one is a long software sequence)
        atomicAdd(&s_hist[e], 1);
      }
    }
    if (valid) {
      if (R == 8) {
        uint64_t packed = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) packed |= (uint64_t)((mask >> d) & 1u) << (8 * d);
        *reinterpret_cast<uint64_t*>(in_rank + (size_t)t * 8) = packed;
      } else {
        for (int d = 0; d < R; ++d) in_rank[(size_t)t * R + d] = (mask >> d) & 1u;
      }
    }
    for (int d = 0; d < R; ++d) {
      const unsigned b = __ballot_sync(0xffffffffu, (mask >> d) & 1u);
      if (lane == 0 && b) atomicAdd(&s_hist[E + d], __popc(b));
    }
  }
  __syncthreads();
  cooperative_groups::this_grid().sync();  // block 0's zeroing is visible
  for (int i = tid; i < E; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&per_expert[i], s_hist[i]);
  for (int i = tid; i < R; i += blockDim.x)
    if (s_hist[E + i]) atomicAdd(&per_rank[i], s_hist[E + i]);
}

constexpr int kClusterBlocks = 16;
constexpr int kClusterThreads = 256;

__global__ void __launch_bounds__(kClusterThreads, 1)
    layout_cluster_kernel(const int64_t* __restrict__ topk_idx, int T, int k, int E, int R,
                          int32_t* __restrict__ per_rank, int32_t* __restrict__ per_expert,
                          uint8_t* __restrict__ in_rank) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ int64_t s_dyn[];
  int64_t* s_topk = s_dyn;                                                        // [blockDim * k]
  int32_t* s_hist = reinterpret_cast<int32_t*>(s_topk + (size_t)blockDim.x * k);  // [E + R]
  const int tid = threadIdx.x, lane = tid & 31;
  const int nb = (int)cluster.num_blocks(), b = (int)cluster.block_rank();
  for (int i = tid; i < E + R; i += blockDim.x) s_hist[i] = 0;
  const int L = E / R;
  for (int t_first = b * blockDim.x; t_first < T; t_first += nb * blockDim.x) {
    const int n_tok = min((int)blockDim.x, T - t_first);
    const int n_words = n_tok * k;
    const int64_t* src = topk_idx + (size_t)t_first * k;
    __syncthreads();
    if (((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (n_words % 2 == 0)) {
      // every 16-byte load of the tile in flight at once (k <= 32: <= 16 per thread)
      constexpr int kPer = 16;
      int4 v[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int i = tid + u * (int)blockDim.x;
        if (i < n_words / 2) v[u] = __ldg(reinterpret_cast<const int4*>(src) + i);
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int i = tid + u * (int)blockDim.x;
        if (i < n_words / 2) reinterpret_cast<int4*>(s_topk)[i] = v[u];
      }
    } else {
      for (int i = tid; i < n_words; i += blockDim.x) s_topk[i] = __ldg(src + i);
    }
    __syncthreads();
    const int t = t_first + tid;
    const bool valid = t < T;
    uint32_t mask = 0;
    for (int j = 0; j < k; ++j) {
      const int64_t e64 = valid ? s_topk[tid * k + j] : -1;
      const int e = (e64 >= 0 && e64 < E) ? (int)e64 : -1;  // out-of-range experts are treated as masked
      if (e >= 0) {
        mask |= 1u << (e / L);
        atomicAdd(&s_hist[e], 1);
      }
    }
    if (valid) {
      if (R == 8) {
        uint64_t packed = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) packed |= (uint64_t)((mask >> d) & 1u) << (8 * d);
        *reinterpret_cast<uint64_t*>(in_rank + (size_t)t * 8) = packed;
      } else {
        for (int d = 0; d < R; ++d) in_rank[(size_t)t * R + d] = (mask >> d) & 1u;
      }
    }
    for (int d = 0; d < R; ++d) {
      const unsigned bal = __ballot_sync(0xffffffffu, (mask >> d) & 1u);
      if (lane == 0 && bal) atomicAdd(&s_hist[E + d], __popc(bal));
    }
  }
  cluster.sync();  // every block's histogram is complete and visible cluster-wide
  // block b sums entries [lo, hi) of the (E + R) histogram over the cluster
  const int n = E + R, lo = (int)((int64_t)n * b / nb), hi = (int)((int64_t)n * (b + 1) / nb);
  for (int i = lo + tid; i < hi; i += blockDim.x) {
    int part[kClusterBlocks];
#pragma unroll
    for (int q = 0; q < kClusterBlocks; ++q) part[q] = q < nb ? cluster.map_shared_rank(s_hist, q)[i] : 0;
    int sum = 0;
#pragma unroll
    for (int q = 0; q < kClusterBlocks; ++q) sum += part[q];
    if (i < E) per_expert[i] = sum;
    else per_rank[i - E] = sum;
  }
  cluster.sync();  // no block leaves while a peer may still read its shared memory
}

}  // namespace epb

using namespace epb;

// Geometry of the normal-mode arena for rows of `hidden` bf16 values and
// `k` top-k entries: num_recv_slots receive slots + 2 (parity) combine
// staging buffers, each holding cap_rows rows.  Identical on every rank.
int compute_recv_layout(const epb_ctx* ctx, int hidden, int k, epb_recv_layout_t* L) {
  if (hidden <= 0 || hidden % 128 != 0) return epb_set_error(EPB_ERR_CONFIG, "hidden must be a positive multiple of 128");
  if (k < 0 || k > 32) return epb_set_error(EPB_ERR_CONFIG, "num_topk must be in [0, 32]");
  const size_t A = 256;
  const size_t S = (size_t)hidden / 128;
  const size_t x_row = 2 * (size_t)hidden;
  const size_t per_row = x_row + S * 4 + (size_t)k * 12 + 4;
  const size_t comb_row = 2 * (size_t)hidden + (size_t)k * 4 + 4;
  const int ns = std::max(1, ctx->cfg.num_recv_slots);
  const int nsend = ctx->cfg.ht_transport == EPB_HT_PROXY ? 1 : 0;  // proxy transport: one send-staging slot
  const size_t overhead = A * (size_t)(6 * (ns + nsend) + 6);
  if (ctx->cfg.nvl_bytes <= overhead) return epb_set_error(EPB_ERR_CONFIG, "num_nvl_bytes too small");
  int64_t cap = (int64_t)((ctx->cfg.nvl_bytes - overhead) / ((ns + nsend) * per_row + 2 * comb_row));
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
  const int64_t comb_bytes =
      align_up(cap * 2 * (size_t)hidden, A) + align_up(cap * (size_t)k * 4, A) + align_up(cap * 4, A);
  L->comb_w_off = align_up(cap * 2 * (size_t)hidden, A);
  L->comb_flag_off = L->comb_w_off + align_up(cap * (size_t)k * 4, A);
  L->comb_off[0] = L->slot0_off + ns * L->slot_bytes;
  L->comb_off[1] = L->comb_off[0] + comb_bytes;
  L->send_off = nsend ? L->comb_off[1] + comb_bytes : 0;
  const int64_t end = nsend ? L->send_off + L->slot_bytes : L->comb_off[1] + comb_bytes;
  if ((size_t)(end - L->slot0_off) > ctx->cfg.nvl_bytes)
    return epb_set_error(EPB_ERR_CONFIG, "internal: recv layout exceeds arena");
  // proxy TransferCmd offsets are 32-bit, relative to the arena start (proxy.cpp)
  if (nsend && (uint64_t)(ctx->ll_off() - epb::kRegionHeader + ctx->cfg.ll_bytes) > 0xFFFFFFFFull)
    return epb_set_error(EPB_ERR_CONFIG, "proxy transport needs num_nvl_bytes + num_rdma_bytes < 4 GiB");
  return EPB_OK;
}

int check_group(epb_t* const* ctxs, int n) {
  if (!ctxs || n <= 0 || n > kMaxLocal) return epb_set_error(EPB_ERR_PROTOCOL, "bad local group");
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i]) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
    for (int r = 0; r < ctxs[i]->world; ++r)
      if (!ctxs[i]->peer[r]) return epb_set_error(EPB_ERR_CONNECTION, "peers not opened");
  }
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
  {
    // one 16-block cluster (B200 opt-in size); refused once -> cooperative fallback
    static int cluster_ok = -1;
    const size_t csmem = sizeof(int64_t) * kClusterThreads * num_topk + sizeof(int32_t) * (num_experts + num_ranks);
    if (cluster_ok != 0 && csmem <= 200 * 1024) {
      cudaError_t e = cudaSuccess;
      if (cluster_ok < 0) {
        e = cudaFuncSetAttribute((const void*)layout_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      }
      // the opt-in limit tracks the real need: a 200 KB limit made the driver
      // give this kernel a different L1/shared split from the dispatch and
      // combine kernels around it, and the SM reconfigured between them
      if (e == cudaSuccess && !std::getenv("EPB_LAYOUT_SMEM_MAX")) e = epb_ensure_smem((const void*)layout_cluster_kernel, csmem);
      else if (e == cudaSuccess && cluster_ok < 0)
        e = cudaFuncSetAttribute((const void*)layout_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024);
      if (e == cudaSuccess) {
        epb_set_carveout((const void*)layout_cluster_kernel, !epb_carveout_skip("layout"));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kClusterBlocks);
        cfg.blockDim = dim3(kClusterThreads);
        cfg.dynamicSmemBytes = csmem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kClusterBlocks;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, layout_cluster_kernel, topk_idx, num_tokens, num_topk, num_experts, num_ranks,
                               num_tokens_per_rank, num_tokens_per_expert, is_token_in_rank);
      }
      if (e == cudaSuccess) {
        cluster_ok = 1;
        return EPB_OK;
      }
      cudaGetLastError();
      cluster_ok = 0;
    }
  }
  static const int threads = [] {
    const char* s = std::getenv("EPB_LAYOUT_THREADS");
    const int v = s ? std::atoi(s) : 128;
    return (v >= 32 && v <= kLayoutThreads && v % 32 == 0) ? v : 128;
  }();
  const size_t smem = sizeof(int64_t) * threads * num_topk + sizeof(int32_t) * (num_experts + num_ranks);
  if (smem > 200 * 1024) return epb_set_error(EPB_ERR_CONFIG, "num_experts too large for layout kernel");
  epb_set_carveout((const void*)layout_kernel, !epb_carveout_skip("layout"));
  EPB_CUDA(epb_ensure_smem((const void*)layout_kernel, smem));
  const int per_sm = std::max(1, epb_max_active_blocks((const void*)layout_kernel, threads, smem));
  int blocks = std::max(1, (num_tokens + threads - 1) / threads);
  static int sms_cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& sms = sms_cache[dev & 63];
  if (sms == 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  blocks = std::min(blocks, per_sm * std::max(1, sms));  // co-resident (grid-stride over token tiles)
  const int64_t* ti = topk_idx;
  int T = num_tokens, k = num_topk, E = num_experts, R = num_ranks;
  void* kargs[] = {(void*)&ti, &T, &k, &E, &R, (void*)&num_tokens_per_rank, (void*)&num_tokens_per_expert,
                   (void*)&is_token_in_rank};
  EPB_CUDA(cudaLaunchCooperativeKernel((const void*)layout_kernel, dim3(blocks), dim3(threads), kargs, smem, st));
  EPB_CUDA(cudaGetLastError());
  return EPB_OK;
}

// Load this file's kernels now (see epb_preload_kernels, api.cpp).
cudaError_t epb_preload_layout() {
  cudaFuncAttributes attr;
  for (const void* fn : {(const void*)layout_kernel, (const void*)layout_cluster_kernel})
    if (cudaError_t e = cudaFuncGetAttributes(&attr, fn)) return e;
  return cudaSuccess;
}
