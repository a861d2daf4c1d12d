// ll.cu — low-latency (decode) EP path on sm_100a, plus the device side of
// the GPU -> CPU command FIFO.
//
//   ll_dispatch : per (token, expert) message, no dedup (SPEC.md:426-434,
//                 :463), fused FP8 e4m3 quantisation per 128 channels,
//                 deterministic slots (rank of the token among the source's
//                 tokens for that expert), one completion signal per source
//                 (the LL fence of PAPER.md:343-346 / kernels.py:187-248
//                 collapses to "all X writes, then the count" because NVLink
//                 stores + release/acquire are ordered).
//   ll_combine  : expert outputs pushed back to the source, weighted top-k
//                 reduce in fp32 in ascending top-k order.
//
// Two transports share the same receive layout:
//   direct : the kernel stores rows into the peer's receive block over NVLink;
//   proxy  : the kernel stores rows into its local send block (same layout)
//            and one producer lane pushes 16-byte TransferCmds (command.py
//            layout) into a pinned-host FIFO (kernels.py:23-31 ctl layout);
//            CPU proxy threads (proxy.cpp) coalesce the WRITEs into copies and
//            execute the piggybacked atomic as a stream-ordered counter bump.
//
// Receive block per (parity, source): [int32 count per local expert, 16-B
// padded][rows in (local expert, ordinal) order].  A row is
// [payload][scales f32 x H/128 (fp8 only)][int32 source token][pad] (16-B
// multiple).  The source knows every row index locally, so no count exchange
// is needed before the data moves.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "ctx.h"

namespace epb {

constexpr int kLLThreads = 256;
constexpr float kFp8Max = 448.0f;

struct LLGeom {
  int R, L, E, k, H, S, Tmax;
  int use_fp8;
  int64_t rows_per_src;
  int64_t disp_row;      // row stride of this call (fp8 or bf16)
  int64_t disp_row_max;  // row stride the region is sized for
  int64_t comb_row;
  int64_t hdr_bytes;
  int64_t disp_block, comb_block;
  int64_t off_disp_recv, off_comb_recv, off_disp_send, off_comb_send;  // from the LL base
  int64_t bytes_needed;
};

static void ll_geometry(int R, int Tmax, int H, int k, int E, int use_fp8, LLGeom* g) {
  std::memset(g, 0, sizeof(*g));
  g->R = R;
  g->E = E;
  g->L = E / R;
  g->k = k;
  g->H = H;
  g->S = H / 128;
  g->Tmax = Tmax;
  g->use_fp8 = use_fp8;
  g->rows_per_src = (int64_t)align_up((size_t)Tmax * std::min(k, g->L), 16);
  const int64_t fp8_row = align_up((size_t)H + 4 * (size_t)g->S + 16, 16);
  const int64_t bf16_row = align_up(2 * (size_t)H + 16, 16);
  g->disp_row_max = std::max(fp8_row, bf16_row);
  g->disp_row = use_fp8 ? fp8_row : bf16_row;
  g->comb_row = 2 * (int64_t)H;
  g->hdr_bytes = align_up(4 * (size_t)g->L, 16);
  g->disp_block = align_up(g->hdr_bytes + g->rows_per_src * g->disp_row_max, 256);
  g->comb_block = align_up(g->rows_per_src * g->comb_row, 256);
  g->off_disp_recv = 0;
  g->off_comb_recv = g->off_disp_recv + 2 * R * g->disp_block;
  g->off_disp_send = g->off_comb_recv + 2 * R * g->comb_block;
  g->off_comb_send = g->off_disp_send + 2 * R * g->disp_block;
  g->bytes_needed = g->off_comb_send + 2 * R * g->comb_block;
}

#ifdef __CUDACC__
// -------------------------------------------------------------------------
// FIFO producer (device side of command_channel.push / check_completion,
// SPEC.md:50-58, :90-98).  Single producer per channel; the tail lives in
// device memory (Scratch), the head is re-read from pinned host memory only
// when the ring looks full.
// -------------------------------------------------------------------------
__device__ __forceinline__ void cmd_pack_dev(uint64_t kind, uint64_t dst, uint64_t ch, uint64_t so, uint64_t dof,
                                             uint64_t len, uint64_t flags, uint64_t& lo, uint64_t& hi) {
  lo = kind | (dst << 2) | (ch << 14) | (so << 20) | ((dof & 0xFFFull) << 52);
  hi = (dof >> 12) | (len << 20) | (flags << 52);
}

__device__ __forceinline__ void st_v2_u64(int64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// Push one command; returns its index or -1 on timeout.
__device__ int64_t fifo_push(const RankView& rv, int ch, uint64_t lo, uint64_t hi) {
  Scratch* sc = scratch_of(rv.base);
  int64_t* ctl = reinterpret_cast<int64_t*>(sc->fifo_ctl[ch]);
  const int64_t cap = sc->fifo_cap;
  const int64_t tail = sc->fifo_tail[ch];
  int64_t head = sc->fifo_head[ch];
  uint64_t t0 = 0;
  while (tail - head >= cap) {  // full: pace on the consumer
    head = ld_acquire_sys(ctl + EPB_CTL_HEAD);
    const uint64_t now = globaltimer();
    if (t0 == 0) t0 = now;
    else if (now - t0 > rv.timeout_ns) {
      report_error(rv, EPB_ERR_DEADLOCK, 0x500 + ch);
      return -1;
    }
  }
  sc->fifo_head[ch] = head;
  st_v2_u64(ctl + EPB_CTL_SLOT0 + 2 * (tail & (cap - 1)), lo, hi);
  st_release_sys(ctl + EPB_CTL_TAIL, tail + 1);
  sc->fifo_tail[ch] = tail + 1;
  return tail;
}

// check_completion(idx): COMPLETED holds the number of commands completed.
__device__ __forceinline__ bool fifo_completed(const RankView& rv, int ch, int64_t idx) {
  int64_t* ctl = reinterpret_cast<int64_t*>(scratch_of(rv.base)->fifo_ctl[ch]);
  return ld_acquire_sys(ctl + EPB_CTL_COMPLETED) > idx;
}

// -------------------------------------------------------------------------
// FP8 e4m3 per-128-channel quantisation of 16 channels held by one lane.
// Eight consecutive lanes own one 128-channel group; amax is reduced over
// them with xor-shuffles.  Formula (pinned in oracle/ep.py:fp8_quant):
//   amax = max(max|x|, 1e-4); scale_inv = amax * (1/448)
//   (round_scale: scale_inv -> 2^ceil(log2 scale_inv)); scale = round ? 1/scale_inv : 448/amax
//   q = cvt.rn.satfinite.e4m3(x * scale)
// -------------------------------------------------------------------------
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ uint16_t cvt_e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ float pow2_ceil(float s) {
  uint32_t u = __float_as_uint(s);
  if (u & 0x7fffffu) u = (u & 0xff800000u) + 0x800000u;
  return __uint_as_float(u & 0xff800000u);
}

// in: two int4 = 16 bf16 channels.  out: 16 e4m3 bytes; returns scale_inv.
__device__ __forceinline__ float quant16(const int4& a, const int4& b, bool active, int round_scale, int4& q) {
  const uint32_t w[8] = {(uint32_t)a.x, (uint32_t)a.y, (uint32_t)a.z, (uint32_t)a.w,
                         (uint32_t)b.x, (uint32_t)b.y, (uint32_t)b.z, (uint32_t)b.w};
  float f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    f[2 * i] = bf16lo(w[i]);
    f[2 * i + 1] = bf16hi(w[i]);
  }
  float amax = 0.0f;
  if (active) {
#pragma unroll
    for (int i = 0; i < 16; ++i) amax = fmaxf(amax, fabsf(f[i]));
  }
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 4));
  amax = fmaxf(amax, 1e-4f);
  float sinv = __fmul_rn(amax, 1.0f / kFp8Max);
  float scale;
  if (round_scale) {
    sinv = pow2_ceil(sinv);
    scale = __fdiv_rn(1.0f, sinv);
  } else {
    scale = __fdiv_rn(kFp8Max, amax);
  }
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t lo = cvt_e4m3x2(__fmul_rn(f[4 * i], scale), __fmul_rn(f[4 * i + 1], scale));
    const uint32_t hi = cvt_e4m3x2(__fmul_rn(f[4 * i + 2], scale), __fmul_rn(f[4 * i + 3], scale));
    o[i] = lo | (hi << 16);
  }
  q = make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]);
  return sinv;
}

// standalone per-token cast (warp per token)
__global__ void __launch_bounds__(kLLThreads) fp8_cast_kernel(const __nv_bfloat16* __restrict__ x, int T, int H,
                                                               int round_scale, uint8_t* __restrict__ q,
                                                               float* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int S = H / 128;
  for (int t = gw; t < T; t += nw) {
    const int4* src = reinterpret_cast<const int4*>(x + (size_t)t * H);
    for (int ch0 = lane * 16; ch0 - lane * 16 < H; ch0 += 512) {
      const bool active = ch0 < H;
      int4 a = make_int4(0, 0, 0, 0), b = a;
      if (active) {
        a = ld_nc_v4(src + ch0 / 8);
        b = ld_nc_v4(src + ch0 / 8 + 1);
      }
      int4 qq;
      const float sinv = quant16(a, b, active, round_scale, qq);
      if (active) {
        *reinterpret_cast<int4*>(q + (size_t)t * H + ch0) = qq;
        if ((lane & 7) == 0) scales[(size_t)t * S + ch0 / 128] = sinv;
      }
    }
  }
}

// -------------------------------------------------------------------------
// LL dispatch
// -------------------------------------------------------------------------
struct LLDispatchParams {
  int n_local, phases, use_proxy, disp_channels;
  uint32_t epoch[kMaxLocal];
  uint64_t proxy_expected[kMaxLocal];
  RankView rv[kMaxLocal];
  epb_ll_dispatch_args_t a[kMaxLocal];
  LLGeom g;
  int64_t ll_off;
};

__device__ __forceinline__ int ordinal_of(const uint32_t* bm_row, int t) {
  const int w = t >> 5;
  int c = 0;
  for (int i = 0; i < w; ++i) c += __popc(bm_row[i]);
  return c + __popc(bm_row[w] & ((1u << (t & 31)) - 1u));
}

__global__ void __launch_bounds__(kLLThreads, 1) ll_dispatch_kernel(const __grid_constant__ LLDispatchParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_ll_dispatch_args_t& a = P.a[lr];
  const LLGeom& g = P.g;
  const int R = g.R, L = g.L, E = g.E, k = g.k, H = g.H, S = g.S, me = rv.rank;
  const int T = a.num_tokens;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const int total_w = gridDim.x * nw;
  const uint32_t epoch = P.epoch[lr];
  const int par = epoch & 1;
  char* my_ll = rv.base + P.ll_off;
  Scratch* sc = scratch_of(rv.base);
  Meta* my_meta = meta_of(rv.base);
  extern __shared__ uint8_t smem[];

  if (P.phases & 1) {
    const int W = max(1, (T + 31) / 32);
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem);
    int32_t* cnt = reinterpret_cast<int32_t*>(bm + (size_t)E * W);
    int32_t* pre = cnt + E;
    uint64_t* dptr = reinterpret_cast<uint64_t*>(smem + align_up(((size_t)E * W + 2 * E) * 4, 16));
    for (int i = tid; i < E * W; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    for (int i = tid; i < T * k; i += blockDim.x) {
      const int64_t e = a.topk_idx[i];
      const int t = i / k;
      if (e >= 0 && e < E) atomicOr(&bm[(size_t)e * W + (t >> 5)], 1u << (t & 31));
    }
    __syncthreads();
    for (int e = tid; e < E; e += blockDim.x) {
      int c = 0;
      for (int w = 0; w < W; ++w) c += __popc(bm[(size_t)e * W + w]);
      cnt[e] = c;
    }
    __syncthreads();
    for (int d = tid; d < R; d += blockDim.x) {
      int run = 0;
      for (int le = 0; le < L; ++le) {
        pre[d * L + le] = run;
        run += cnt[d * L + le];
      }
    }
    __syncthreads();

    const int64_t rstride = g.disp_row;
    const int meta_off = g.use_fp8 ? H + 4 * S : 2 * H;
    for (int t = blockIdx.x * nw + warp; t < T; t += total_w) {
      if (lane < k) {
        const int64_t e = a.topk_idx[(size_t)t * k + lane];
        uint64_t p = 0;
        int32_t slot = -1;
        if (e >= 0 && e < E) {
          const int d = (int)(e / L);
          const int row = pre[e] + ordinal_of(bm + (size_t)e * W, t);
          char* blk = P.use_proxy ? my_ll + g.off_disp_send + (int64_t)(par * R + d) * g.disp_block
                                  : rv.peer[d] + P.ll_off + g.off_disp_recv + (int64_t)(par * R + me) * g.disp_block;
          p = reinterpret_cast<uint64_t>(blk + g.hdr_bytes + (int64_t)row * rstride);
          slot = (int32_t)(d * g.rows_per_src + row);
        }
        dptr[warp * k + lane] = p;
        a.comb_slot[(size_t)t * k + lane] = slot;
      }
      __syncwarp();
      const int4* src = reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + (size_t)t * H * 2);
      if (g.use_fp8) {
        for (int ch0 = lane * 16; ch0 - lane * 16 < H; ch0 += 512) {
          const bool active = ch0 < H;
          int4 x0 = make_int4(0, 0, 0, 0), x1 = x0;
          if (active) {
            x0 = ld_nc_v4(src + ch0 / 8);
            x1 = ld_nc_v4(src + ch0 / 8 + 1);
          }
          int4 q;
          const float sinv = quant16(x0, x1, active, a.round_scale, q);
          if (active) {
            for (int j = 0; j < k; ++j) {
              char* p = reinterpret_cast<char*>(dptr[warp * k + j]);
              if (p == nullptr) continue;
              st_v4(reinterpret_cast<int4*>(p + ch0), q);
              if ((lane & 7) == 0) reinterpret_cast<float*>(p + H)[ch0 / 128] = sinv;
            }
          }
        }
      } else {
        const int n16 = H / 8;
        for (int i = lane; i < n16; i += 32) {
          const int4 v = ld_nc_v4(src + i);
          for (int j = 0; j < k; ++j) {
            char* p = reinterpret_cast<char*>(dptr[warp * k + j]);
            if (p != nullptr) st_v4(reinterpret_cast<int4*>(p) + i, v);
          }
        }
      }
      if (lane < k) {
        char* p = reinterpret_cast<char*>(dptr[warp * k + lane]);
        if (p != nullptr) *reinterpret_cast<int32_t*>(p + meta_off) = t;
      }
      __syncwarp();
    }

    // last warp of this rank publishes the per-expert counts and the signal
    fence_sys();
    __syncwarp();
    uint32_t last = 0;
    if (lane == 0) last = atomicAdd(&sc->ll_ticket[par], 1u) == (uint32_t)(total_w - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      if (lane == 0) sc->ll_ticket[par] = 0;
      for (int d = 0; d < R; ++d) {
        char* blk = P.use_proxy ? my_ll + g.off_disp_send + (int64_t)(par * R + d) * g.disp_block
                                : rv.peer[d] + P.ll_off + g.off_disp_recv + (int64_t)(par * R + me) * g.disp_block;
        for (int le = lane; le < L; le += 32) reinterpret_cast<int32_t*>(blk)[le] = cnt[d * L + le];
      }
      fence_sys();
      __syncwarp();
      if (!P.use_proxy) {
        if (lane < R) st_release_sys(&meta_of(rv.peer[lane])->ll_disp_flag[par][me], (uint64_t)epoch);
      } else if (lane == 0) {
        for (int d = 0; d < R; ++d) {
          int rows = 0;
          for (int le = 0; le < L; ++le) rows += cnt[d * L + le];
          const int ch = d % P.disp_channels;
          const int64_t src_off = g.off_disp_send + (int64_t)(par * R + d) * g.disp_block;
          const int64_t dst_off = g.off_disp_recv + (int64_t)(par * R + me) * g.disp_block;
          const int64_t len = g.hdr_bytes + (int64_t)rows * rstride;
          uint64_t lo, hi;
          cmd_pack_dev(EPB_CMD_WRITE, d, ch, src_off, dst_off, len, EPB_FLAG_PIGGYBACK_ATOMIC, lo, hi);
          fifo_push(rv, ch, lo, hi);
        }
      }
    }
  }

  if (P.phases & 2) {
    // receive: wait for every source, then compact into the packed layout
    int32_t* s_hdr = reinterpret_cast<int32_t*>(smem);   // [R][L]
    int32_t* s_off = s_hdr + R * L;                       // [R][L] prefix over sources
    int32_t* s_pre = s_off + R * L;                       // [R][L] prefix over experts (row in block)
    int32_t* s_tot = s_pre + R * L;                       // [L + 1] prefix over experts of totals
    if (tid < R) {
      if (!P.use_proxy) wait_geq64(rv, &my_meta->ll_disp_flag[par][tid], (uint64_t)epoch, 0x600 + tid);
      else wait_geq64(rv, &my_meta->proxy_sig[me % P.disp_channels][tid], P.proxy_expected[lr], 0x680 + tid);
    }
    __syncthreads();
    for (int i = tid; i < R * L; i += blockDim.x) {
      const int s = i / L, le = i % L;
      s_hdr[i] = __ldcg(reinterpret_cast<const int32_t*>(my_ll + g.off_disp_recv +
                                                          (int64_t)(par * R + s) * g.disp_block) + le);
    }
    __syncthreads();
    for (int le = tid; le < L; le += blockDim.x) {
      int run = 0;
      for (int s = 0; s < R; ++s) {
        s_off[s * L + le] = run;
        run += s_hdr[s * L + le];
      }
      s_tot[le + 1] = run;
    }
    for (int s = tid; s < R; s += blockDim.x) {
      int run = 0;
      for (int le = 0; le < L; ++le) {
        s_pre[s * L + le] = run;
        run += s_hdr[s * L + le];
      }
    }
    __syncthreads();
    if (tid == 0) {
      s_tot[0] = 0;
      for (int le = 0; le < L; ++le) s_tot[le + 1] += s_tot[le];
    }
    __syncthreads();
    const int RT = R * g.Tmax;
    if (blockIdx.x == 0) {
      for (int le = tid; le < L; le += blockDim.x) a.packed_recv_count[le] = s_tot[le + 1] - s_tot[le];
      for (int i = tid; i < R * L; i += blockDim.x) {
        const int le = i / R, s = i % R;
        a.packed_recv_layout_range[i] = ((int64_t)s_off[s * L + le] << 32) | (int64_t)s_hdr[s * L + le];
      }
    }
    const int N = s_tot[L];
    const int64_t rstride = g.disp_row;
    const int meta_off = g.use_fp8 ? H + 4 * S : 2 * H;
    const int pay16 = g.use_fp8 ? H / 16 : H / 8;
    for (int item = blockIdx.x * nw + warp; item < N; item += total_w) {
      int lo = 0, hi = L;  // find le: s_tot[le] <= item < s_tot[le+1]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_tot[mid] <= item) lo = mid; else hi = mid;
      }
      const int le = lo, j = item - s_tot[le];
      int s = 0;
      while (s < R - 1 && j >= s_off[s * L + le] + s_hdr[s * L + le]) ++s;
      const int row = s_pre[s * L + le] + (j - s_off[s * L + le]);
      const char* rp = my_ll + g.off_disp_recv + (int64_t)(par * R + s) * g.disp_block + g.hdr_bytes + row * rstride;
      const int4* src = reinterpret_cast<const int4*>(rp);
      int4* dst = reinterpret_cast<int4*>(static_cast<char*>(a.packed_recv_x) +
                                          ((int64_t)le * RT + j) * (g.use_fp8 ? H : 2 * H));
      for (int i = lane; i < pay16; i += 32) st_na_v4(dst + i, ld_cg_v4(src + i));
      if (g.use_fp8 && a.packed_recv_x_scales != nullptr)
        for (int q = lane; q < S; q += 32)
          a.packed_recv_x_scales[((int64_t)le * S + q) * RT + j] = __ldcg(reinterpret_cast<const float*>(rp + H) + q);
      if (lane == 0) {
        a.packed_recv_src_info[(int64_t)le * RT + j] = __ldcg(reinterpret_cast<const int32_t*>(rp + meta_off));
        a.recv_route[(int64_t)le * RT + j] = (int32_t)(s * g.rows_per_src + row);
      }
    }
  }
}

// -------------------------------------------------------------------------
// LL combine
// -------------------------------------------------------------------------
struct LLCombineParams {
  int n_local, phases, use_proxy, disp_channels;
  uint32_t epoch[kMaxLocal];
  uint64_t proxy_expected[kMaxLocal];
  RankView rv[kMaxLocal];
  epb_ll_combine_args_t a[kMaxLocal];
  LLGeom g;
  int64_t ll_off;
};

__global__ void __launch_bounds__(kLLThreads, 1) ll_combine_kernel(const __grid_constant__ LLCombineParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_ll_combine_args_t& a = P.a[lr];
  const LLGeom& g = P.g;
  const int R = g.R, L = g.L, H = g.H, me = rv.rank, k = g.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const int total_w = gridDim.x * nw;
  const uint32_t epoch = P.epoch[lr];
  const int par = epoch & 1;
  char* my_ll = rv.base + P.ll_off;
  Scratch* sc = scratch_of(rv.base);
  Meta* my_meta = meta_of(rv.base);
  const int RT = R * g.Tmax;
  const int n16 = H / 8;
  __shared__ int32_t s_tot[kMaxLocalExperts + 1];

  if (P.phases & 1) {
    if (tid == 0) {
      s_tot[0] = 0;
      for (int le = 0; le < L; ++le) s_tot[le + 1] = s_tot[le] + a.packed_recv_count[le];
    }
    __syncthreads();
    const int N = s_tot[L];
    for (int item = blockIdx.x * nw + warp; item < N; item += total_w) {
      int lo = 0, hi = L;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_tot[mid] <= item) lo = mid; else hi = mid;
      }
      const int le = lo, j = item - s_tot[le];
      const int route = a.recv_route[(int64_t)le * RT + j];
      const int s = (int)(route / g.rows_per_src), row = (int)(route % g.rows_per_src);
      char* blk = P.use_proxy ? my_ll + g.off_comb_send + (int64_t)(par * R + s) * g.comb_block
                              : rv.peer[s] + P.ll_off + g.off_comb_recv + (int64_t)(par * R + me) * g.comb_block;
      int4* dst = reinterpret_cast<int4*>(blk + (int64_t)row * g.comb_row);
      const int4* src = reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + ((int64_t)le * RT + j) * 2 * H);
      for (int i = lane; i < n16; i += 32) st_v4(dst + i, ld_nc_v4(src + i));
    }
    fence_sys();
    __syncwarp();
    uint32_t last = 0;
    if (lane == 0) last = atomicAdd(&sc->ll_ticket[2 + par], 1u) == (uint32_t)(total_w - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      if (lane == 0) sc->ll_ticket[2 + par] = 0;
      if (!P.use_proxy) {
        if (lane < R) st_release_sys(&meta_of(rv.peer[lane])->ll_comb_flag[par][me], (uint64_t)epoch);
      } else if (lane == 0) {
        for (int s = 0; s < R; ++s) {
          int64_t rows = 0;
          for (int le = 0; le < L; ++le) rows += a.packed_recv_layout_range[le * R + s] & 0xffffffffll;
          const int ch = P.disp_channels + s % P.disp_channels;
          const int64_t src_off = g.off_comb_send + (int64_t)(par * R + s) * g.comb_block;
          const int64_t dst_off = g.off_comb_recv + (int64_t)(par * R + me) * g.comb_block;
          uint64_t lo, hi;
          cmd_pack_dev(EPB_CMD_WRITE, s, ch, src_off, dst_off, rows * g.comb_row, EPB_FLAG_PIGGYBACK_ATOMIC, lo, hi);
          fifo_push(rv, ch, lo, hi);
        }
      }
    }
  }

  if (P.phases & 2) {
    if (tid < R) {
      if (!P.use_proxy) wait_geq64(rv, &my_meta->ll_comb_flag[par][tid], (uint64_t)epoch, 0x700 + tid);
      else wait_geq64(rv, &my_meta->proxy_sig[P.disp_channels + me % P.disp_channels][tid], P.proxy_expected[lr],
                      0x780 + tid);
    }
    __syncthreads();
    const int T = a.num_tokens;
    for (int t = blockIdx.x * nw + warp; t < T; t += total_w) {
      const int4* rows[32];
      float w[32];
      for (int j = 0; j < k; ++j) {
        const int slot = a.comb_slot[(size_t)t * k + j];
        if (slot >= 0) {
          const int r = (int)(slot / g.rows_per_src), row = (int)(slot % g.rows_per_src);
          rows[j] = reinterpret_cast<const int4*>(my_ll + g.off_comb_recv + (int64_t)(par * R + r) * g.comb_block +
                                                  (int64_t)row * g.comb_row);
          w[j] = a.topk_weights[(size_t)t * k + j];
        } else {
          rows[j] = nullptr;
          w[j] = 0.0f;
        }
      }
      int4* out = reinterpret_cast<int4*>(static_cast<char*>(a.combined_x) + (size_t)t * H * 2);
      for (int i = lane; i < n16; i += 32) {
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
        for (int j = 0; j < k; ++j) {
          if (rows[j] == nullptr) continue;
          const int4 v = ld_cg_v4(rows[j] + i);
          const uint32_t u[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[2 * q] = __fadd_rn(acc[2 * q], __fmul_rn(w[j], bf16lo(u[q])));
            acc[2 * q + 1] = __fadd_rn(acc[2 * q + 1], __fmul_rn(w[j], bf16hi(u[q])));
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
    }
  }
}

// -------------------------------------------------------------------------
// FIFO microbench: one producer warp per channel pushes WRITE commands in
// batches of 32 slots (one 512-B burst over PCIe, one tail publish), then
// waits until the proxy reports them completed (check_completion).
// -------------------------------------------------------------------------
__global__ void fifo_bench_kernel(RankView rv, int64_t n_per_ch, int channels, int64_t* elapsed) {
  const int ch = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (ch >= channels) return;
  Scratch* sc = scratch_of(rv.base);
  int64_t* ctl = reinterpret_cast<int64_t*>(sc->fifo_ctl[ch]);
  const int64_t cap = sc->fifo_cap;
  int64_t tail = sc->fifo_tail[ch], head = sc->fifo_head[ch];
  const int64_t start = tail, end = tail + n_per_ch;
  const uint64_t t0 = globaltimer();
  bool ok = true;
  while (tail < end && ok) {
    const int64_t n = min((int64_t)32, min(end - tail, cap));
    uint64_t ts = 0;
    while (tail + n - head > cap) {
      head = ld_acquire_sys(ctl + EPB_CTL_HEAD);
      const uint64_t now = globaltimer();
      if (ts == 0) ts = now;
      else if (now - ts > rv.timeout_ns) {
        if (lane == 0) report_error(rv, EPB_ERR_DEADLOCK, 0x800 + ch);
        ok = false;
        break;
      }
    }
    if (!ok) break;
    if (lane < n) {
      uint64_t lo, hi;
      const int64_t idx = tail + lane;
      cmd_pack_dev(EPB_CMD_WRITE, 0, ch, (uint64_t)(idx & 0xffffffff), 0, 0, 0, lo, hi);
      st_v2_u64(ctl + EPB_CTL_SLOT0 + 2 * (idx & (cap - 1)), lo, hi);
    }
    fence_sys();
    __syncwarp();
    tail += n;
    if (lane == 0) st_release_sys(ctl + EPB_CTL_TAIL, tail);
  }
  if (ok && lane == 0) {
    uint64_t ts = globaltimer();
    while (!fifo_completed(rv, ch, end - 1)) {
      if (globaltimer() - ts > rv.timeout_ns) {
        report_error(rv, EPB_ERR_DEADLOCK, 0x900 + ch);
        break;
      }
    }
  }
  if (lane == 0) {
    sc->fifo_tail[ch] = tail;
    sc->fifo_head[ch] = head;
    atomicMax(reinterpret_cast<unsigned long long*>(elapsed), (unsigned long long)(globaltimer() - t0));
  }
  (void)start;
}
#endif  // __CUDACC__

}  // namespace epb

using namespace epb;

extern "C" int epb_ll_layout(int num_ranks, int max_tokens, int hidden, int num_topk, int num_experts, int use_fp8,
                             epb_ll_layout_t* out) {
  if (!out) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  if (num_ranks <= 0 || num_ranks > kMaxRanks || num_experts <= 0 || num_experts % num_ranks)
    return epb_set_error(EPB_ERR_CONFIG, "num_experts must be a positive multiple of num_ranks (<= 8 ranks)");
  if (hidden <= 0 || hidden % 128) return epb_set_error(EPB_ERR_CONFIG, "hidden must be a multiple of 128");
  if (num_topk <= 0 || num_topk > 32) return epb_set_error(EPB_ERR_CONFIG, "num_topk must be in [1, 32]");
  if (max_tokens <= 0) return epb_set_error(EPB_ERR_CONFIG, "max_tokens must be positive");
  LLGeom g;
  ll_geometry(num_ranks, max_tokens, hidden, num_topk, num_experts, use_fp8, &g);
  out->rows_per_src = g.rows_per_src;
  out->disp_row_bytes = g.disp_row;
  out->comb_row_bytes = g.comb_row;
  out->bytes_needed = g.bytes_needed;
  return EPB_OK;
}

static int ll_check(epb_ctx* c, const LLGeom& g) {
  if ((size_t)g.bytes_needed > c->cfg.ll_bytes)
    return epb_set_error(EPB_ERR_CONFIG, "low-latency region too small: need " + std::to_string(g.bytes_needed) +
                                             " bytes, have " + std::to_string(c->cfg.ll_bytes));
  if (g.E / g.R > kMaxLocalExperts) return epb_set_error(EPB_ERR_CONFIG, "too many local experts");
  return EPB_OK;
}

static int check_group_ll(epb_t* const* ctxs, int n) {
  if (!ctxs || n <= 0 || n > kMaxLocal) return epb_set_error(EPB_ERR_PROTOCOL, "bad local group");
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i]) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
    for (int r = 0; r < ctxs[i]->world; ++r)
      if (!ctxs[i]->peer[r]) return epb_set_error(EPB_ERR_CONNECTION, "peers not opened");
  }
  return EPB_OK;
}

static int ll_blocks(epb_t* const* ctxs, int n_local, int num_sms, const void* kernel, size_t smem) {
  int max_active = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_active, kernel, kLLThreads, smem) != cudaSuccess ||
      max_active < 1)
    max_active = 1;
  int nb = std::max(1, num_sms / n_local);
  return std::min(nb, std::max(1, max_active * ctxs[0]->num_sms / n_local));
}

extern "C" int epb_ll_dispatch(epb_t* const* ctxs, int n_local, const epb_ll_dispatch_args_t* args, int num_sms,
                               void* stream) {
  if (int e = check_group_ll(ctxs, n_local)) return e;
  LLDispatchParams P;
  std::memset(&P, 0, sizeof(P));
  const epb_ll_dispatch_args_t& a0 = args[0];
  if (a0.num_tokens > a0.max_tokens) return epb_set_error(EPB_ERR_CONFIG, "num_tokens exceeds num_max_dispatch_tokens_per_rank");
  ll_geometry(ctxs[0]->world, a0.max_tokens, a0.hidden, a0.num_topk, a0.num_experts, a0.use_fp8, &P.g);
  P.n_local = n_local;
  P.phases = a0.phases;
  P.use_proxy = a0.use_proxy;
  P.ll_off = (int64_t)ctxs[0]->ll_off();
  if (P.phases < 1 || P.phases > 3) return epb_set_error(EPB_ERR_PROTOCOL, "phases must be 1, 2 or 3");
  for (int i = 0; i < n_local; ++i) {
    epb_ctx* c = ctxs[i];
    if (int e = ll_check(c, P.g)) return e;
    if (args[i].num_tokens > args[i].max_tokens) return epb_set_error(EPB_ERR_CONFIG, "num_tokens exceeds max_tokens");
    if (P.use_proxy) {
      if (c->cfg.fifo_channels < 2 || !c->proxy)
        return epb_set_error(EPB_ERR_UNSUPPORTED, "proxy transport needs >= 2 FIFO channels and a running proxy");
      P.disp_channels = c->cfg.fifo_channels / 2;
    } else {
      P.disp_channels = std::max(1, c->cfg.fifo_channels / 2);
    }
    if (P.phases & 1) {
      ++c->ll_disp_epoch;
      if (P.use_proxy) ++c->ll_proxy_disp;
    }
    P.epoch[i] = c->ll_disp_epoch;
    P.proxy_expected[i] = c->ll_proxy_disp;
    P.rv[i] = c->view();
    P.a[i] = args[i];
  }
  const int W = std::max(1, (a0.max_tokens + 31) / 32);
  size_t smem_send = align_up(((size_t)P.g.E * W + 2 * P.g.E) * 4, 16) + (size_t)(kLLThreads / 32) * P.g.k * 8;
  size_t smem_recv = (size_t)(3 * P.g.R * P.g.L + P.g.L + 1) * 4;
  size_t smem = std::max(smem_send, smem_recv);
  if (smem > 200 * 1024) return epb_set_error(EPB_ERR_CONFIG, "LL dispatch shape needs too much shared memory");
  if (smem > 48 * 1024)
    EPB_CUDA(cudaFuncSetAttribute(ll_dispatch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int nb = ll_blocks(ctxs, n_local, num_sms, (const void*)ll_dispatch_kernel, smem);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(cudaLaunchCooperativeKernel((void*)ll_dispatch_kernel, dim3(nb, n_local), dim3(kLLThreads), kargs, smem, st));
  return EPB_OK;
}

extern "C" int epb_ll_combine(epb_t* const* ctxs, int n_local, const epb_ll_combine_args_t* args, int num_sms,
                              void* stream) {
  if (int e = check_group_ll(ctxs, n_local)) return e;
  LLCombineParams P;
  std::memset(&P, 0, sizeof(P));
  const epb_ll_combine_args_t& a0 = args[0];
  ll_geometry(ctxs[0]->world, a0.max_tokens, a0.hidden, a0.num_topk, a0.num_experts, 0, &P.g);
  P.n_local = n_local;
  P.phases = a0.phases;
  P.use_proxy = a0.use_proxy;
  P.ll_off = (int64_t)ctxs[0]->ll_off();
  if (P.phases < 1 || P.phases > 3) return epb_set_error(EPB_ERR_PROTOCOL, "phases must be 1, 2 or 3");
  if (P.g.k > 32) return epb_set_error(EPB_ERR_CONFIG, "num_topk must be <= 32");
  for (int i = 0; i < n_local; ++i) {
    epb_ctx* c = ctxs[i];
    if (int e = ll_check(c, P.g)) return e;
    if (P.use_proxy) {
      if (c->cfg.fifo_channels < 2 || !c->proxy)
        return epb_set_error(EPB_ERR_UNSUPPORTED, "proxy transport needs >= 2 FIFO channels and a running proxy");
      P.disp_channels = c->cfg.fifo_channels / 2;
    } else {
      P.disp_channels = std::max(1, c->cfg.fifo_channels / 2);
    }
    if (P.phases & 1) {
      ++c->ll_comb_epoch;
      if (P.use_proxy) ++c->ll_proxy_comb;
    }
    P.epoch[i] = c->ll_comb_epoch;
    P.proxy_expected[i] = c->ll_proxy_comb;
    P.rv[i] = c->view();
    P.a[i] = args[i];
  }
  const int nb = ll_blocks(ctxs, n_local, num_sms, (const void*)ll_combine_kernel, 0);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(cudaLaunchCooperativeKernel((void*)ll_combine_kernel, dim3(nb, n_local), dim3(kLLThreads), kargs, 0, st));
  return EPB_OK;
}

extern "C" int epb_per_token_cast_to_fp8(const void* x, int num_tokens, int hidden, int round_scale, void* q,
                                         float* scales, void* stream) {
  if (hidden <= 0 || hidden % 128) return epb_set_error(EPB_ERR_CONFIG, "hidden must be a multiple of 128");
  if (num_tokens <= 0) return EPB_OK;
  const int warps_per_block = kLLThreads / 32;
  const int blocks = std::min(4096, (num_tokens + warps_per_block - 1) / warps_per_block);
  fp8_cast_kernel<<<blocks, kLLThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), num_tokens, hidden, round_scale, static_cast<uint8_t*>(q), scales);
  EPB_CUDA(cudaGetLastError());
  return EPB_OK;
}

int epb_proxy_set_count_only(epb_ctx* ctx, bool on);  // proxy.cpp

extern "C" int epb_fifo_device_bench(epb_t* ctx, int64_t num_cmds, int channels, int64_t* elapsed_ns, void* stream) {
  if (!ctx || !elapsed_ns) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  if (channels <= 0 || channels > ctx->cfg.fifo_channels || channels > 32)
    return epb_set_error(EPB_ERR_CONFIG, "channels must be in [1, min(32, fifo_channels)]");
  if (!ctx->proxy) return epb_set_error(EPB_ERR_UNSUPPORTED, "proxy not running");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* d_el = nullptr;
  EPB_CUDA(cudaMallocAsync(&d_el, sizeof(int64_t), st));
  EPB_CUDA(cudaMemsetAsync(d_el, 0, sizeof(int64_t), st));
  epb_proxy_set_count_only(ctx, true);
  fifo_bench_kernel<<<1, 32 * channels, 0, st>>>(ctx->view(), num_cmds / channels, channels, d_el);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(elapsed_ns, d_el, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  epb_proxy_set_count_only(ctx, false);
  cudaFreeAsync(d_el, st);
  if (e != cudaSuccess) return epb_cuda_check(e, "fifo_device_bench");
  if (ctx->host->err_code) return epb_set_error((int)ctx->host->err_code, "device FIFO bench reported an error");
  return EPB_OK;
}
