// ll_common.cuh — geometry of the low-latency region, the device side of the
// GPU -> CPU command FIFO, and the FP8 e4m3 per-128-channel quantiser.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace epb {

// 8 warps per block.  (512-thread blocks fill the register file; the proxy
// transport's same-device copies then could not make progress in the 1-GPU
// emulated tests, so the LL grid leaves the SMs room to co-schedule them.)
constexpr int kLLThreads = 256;
constexpr float kFp8Max = 448.0f;

// Low-latency region of one rank (offsets from the LL base, identical on all ranks):
//   disp_recv[2 parity][R src]  blocks: [int32 count per local expert, 16-B padded][rows]
//   comb_recv[2][R src]         blocks: [rows] (mirror of what this rank dispatched to src)
//   disp_send[2][R dst], comb_send[2][R dst]: same layouts, used by the proxy transport
// A dispatch row is [payload][f32 scales x H/128 (fp8 only)][int32 source token][pad to 16 B].
struct LLGeom {
  int R, L, E, k, H, S, Tmax;
  int use_fp8;
  int64_t rows_per_src;
  int64_t disp_row;      // row stride of this call (fp8 or bf16)
  int64_t disp_row_max;  // row stride the region is sized for
  int64_t comb_row;
  int64_t hdr_bytes;
  int64_t disp_block, comb_block;
  int64_t off_disp_recv, off_comb_recv, off_disp_send, off_comb_send;
  int64_t bytes_needed;
};

inline void ll_geometry(int R, int Tmax, int H, int k, int E, int use_fp8, LLGeom* g) {
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
// ---------------------------------------------------------------------------
// FIFO producer (device side of command_channel.push / check_completion,
// SPEC.md:50-58, :90-98).  Single producer per channel; the tail lives in
// device memory (Scratch), the head is re-read from pinned host memory only
// when the ring looks full.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cmd_pack_dev(uint64_t kind, uint64_t dst, uint64_t ch, uint64_t so, uint64_t dof,
                                             uint64_t len, uint64_t flags, uint64_t& lo, uint64_t& hi) {
  lo = kind | (dst << 2) | (ch << 14) | (so << 20) | ((dof & 0xFFFull) << 52);
  hi = (dof >> 12) | (len << 20) | (flags << 52);
}

__device__ __forceinline__ void st_v2_u64(int64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// Push one command; returns its index or -1 on timeout.
__device__ inline int64_t fifo_push(const RankView& rv, int ch, uint64_t lo, uint64_t hi) {
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

// ---------------------------------------------------------------------------
// FP8 e4m3 per-128-channel quantisation of 16 channels held by one lane.
// Eight consecutive lanes own one 128-channel group; amax is reduced over
// them with xor-shuffles.  Formula (pinned in oracle/ep.py:fp8_quant):
//   amax = max(max|x|, 1e-4); scale_inv = amax * (1/448)
//   (round_scale: scale_inv -> 2^ceil(log2 scale_inv)); scale = round ? 1/scale_inv : 448/amax
//   q = cvt.rn.satfinite.e4m3(x * scale)
// ---------------------------------------------------------------------------
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
// Must be called by all 32 lanes (shuffles).
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
#endif  // __CUDACC__

}  // namespace epb
