// fifo.cu — device-side FIFO microbenchmark (SPEC.md:513-521 fifo_stress with
// a GPU producer): one producer warp per channel pushes WRITE commands in
// batches of 32 slots (one 512-B burst over PCIe/C2C, one tail publish), then
// waits until the proxy reports them completed (check_completion).
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <ctime>

#include "ctx.h"
#include "ll_common.cuh"

namespace epb {

// The proxy's SM copy engine (epb_pcopy_batch, ctx.h): blocks [block0, block0 +
// blocks) of a job split each of its segments into contiguous 16-byte ranges
// (ld.global.nc + plain stores, over NVLink for a peer destination); the last
// block of the job (a ticket) publishes its signal with st.release.sys after a
// fence that orders every block's copies (release fence + relaxed RMW pattern).
__global__ void __launch_bounds__(512) pcopy_kernel(const __grid_constant__ epb_pcopy_batch B) {
  if (B.stamp != nullptr && threadIdx.x == 0) {
    const unsigned long long now = globaltimer();
    if (blockIdx.x == 0) B.stamp[0] = (int64_t)now;
    atomicMax(reinterpret_cast<unsigned long long*>(&B.stamp[2]), now);  // the last block to start
  }
  int j = 0;
  while (j + 1 < B.njobs && (int)blockIdx.x >= B.jobs[j + 1].block0) ++j;
  const epb_pcopy_job& J = B.jobs[j];
  const int bj = blockIdx.x - J.block0, nbj = J.blocks;
  for (int s = J.seg0; s < J.seg0 + J.nseg; ++s) {
    const epb_pcopy_seg& g = B.segs[s];
    if (((reinterpret_cast<uintptr_t>(g.src) | reinterpret_cast<uintptr_t>(g.dst)) & 15) != 0) {
      // unaligned segment (e.g. a weights array): bytes, strided over the job's blocks
      for (uint64_t i = (uint64_t)bj * blockDim.x + threadIdx.x; i < g.len; i += (uint64_t)nbj * blockDim.x)
        g.dst[i] = g.src[i];
      continue;
    }
    const uint64_t n16 = g.len >> 4;
    const uint64_t u0 = n16 * bj / nbj, u1 = n16 * (bj + 1) / nbj;
    const int4* src = reinterpret_cast<const int4*>(g.src);
    int4* dst = reinterpret_cast<int4*>(g.dst);
    uint64_t u = u0 + threadIdx.x;
    for (; u + 3 * blockDim.x < u1; u += 4 * blockDim.x) {
      const int4 v0 = ld_nc_v4(src + u), v1 = ld_nc_v4(src + u + blockDim.x);
      const int4 v2 = ld_nc_v4(src + u + 2 * blockDim.x), v3 = ld_nc_v4(src + u + 3 * blockDim.x);
      st_v4(dst + u, v0);
      st_v4(dst + u + blockDim.x, v1);
      st_v4(dst + u + 2 * blockDim.x, v2);
      st_v4(dst + u + 3 * blockDim.x, v3);
    }
    for (; u < u1; u += blockDim.x) st_v4(dst + u, ld_nc_v4(src + u));
    if (bj == nbj - 1 && threadIdx.x < (g.len & 15))  // tail bytes
      g.dst[(n16 << 4) + threadIdx.x] = g.src[(n16 << 4) + threadIdx.x];
  }
  if (J.sig == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (B.stamp != nullptr) atomicMax(reinterpret_cast<unsigned long long*>(&B.stamp[3]), (unsigned long long)globaltimer());
    fence_sys();
    if (atomicAdd(&B.tickets[j], 1u) == (uint32_t)nbj - 1) {
      B.tickets[j] = 0;
      fence_sys();
      st_release_sys(J.sig, J.sig_val);
      if (B.stamp != nullptr) atomicMax(reinterpret_cast<unsigned long long*>(&B.stamp[1]), (unsigned long long)globaltimer());
    }
  }
}

__global__ void fifo_bench_kernel(RankView rv, int64_t n_per_ch, int channels, int64_t* elapsed) {
  const int ch = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (ch >= channels) return;
  Scratch* sc = scratch_of(rv.base);
  int64_t* ctl = reinterpret_cast<int64_t*>(sc->fifo_ctl[ch]);
  const int64_t cap = sc->fifo_cap;
  int64_t tail = sc->fifo_tail[ch], head = sc->fifo_head[ch];
  const int64_t end = tail + n_per_ch;
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
    const uint64_t ts = globaltimer();
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
}

// Barrier through the proxy (Barrier is blocking on the
// GPU side): push one BARRIER command and spin on check_completion(idx).
__global__ void proxy_barrier_kernel(RankView rv, int ch, int same_rail) {
  if (threadIdx.x != 0) return;
  uint64_t lo, hi;
  cmd_pack_dev(EPB_CMD_BARRIER, (uint64_t)rv.rank, (uint64_t)ch, 0, 0, 0,
               same_rail ? EPB_FLAG_SAME_RAIL_BARRIER : 0, lo, hi);
  const int64_t idx = fifo_push(rv, ch, lo, hi);
  if (idx < 0) return;
  uint64_t t0 = 0;
  int iter = 0;
  while (!fifo_completed(rv, ch, idx)) {
    if ((++iter & 255) == 0) {
      const uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > rv.timeout_ns) {
        report_error(rv, EPB_ERR_DEADLOCK, 0xa00 + ch);
        return;
      }
    }
  }
}

}  // namespace epb

using namespace epb;

extern "C" int epb_proxy_barrier(epb_t* ctx, int channel, int same_rail, void* stream) {
  if (!ctx) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
  if (channel < 0 || channel >= ctx->cfg.fifo_channels) return epb_set_error(EPB_ERR_CONFIG, "no such FIFO channel");
  if (!ctx->proxy) return epb_set_error(EPB_ERR_UNSUPPORTED, "proxy not running");
  proxy_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(ctx->view(), channel, same_rail);
  EPB_CUDA(cudaGetLastError());
  return EPB_OK;
}

namespace epb {
// Drain(Idx): push DRAIN with length_or_value = Idx + 1 (0 = everything) and
// block until check_completion(its index).
__device__ __forceinline__ bool drain_and_wait(const RankView& rv, int ch, int64_t upto) {
  uint64_t lo, hi;
  cmd_pack_dev(EPB_CMD_DRAIN, (uint64_t)rv.rank, (uint64_t)ch, 0, 0, upto < 0 ? 0 : (uint64_t)(upto + 1), 0, lo, hi);
  const int64_t idx = fifo_push(rv, ch, lo, hi);
  if (idx < 0) return false;
  uint64_t t0 = 0;
  int iter = 0;
  while (!fifo_completed(rv, ch, idx)) {
    if ((++iter & 255) == 0) {
      const uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > rv.timeout_ns) {
        report_error(rv, EPB_ERR_DEADLOCK, 0xb00 + ch);
        return false;
      }
    }
  }
  return true;
}

__global__ void proxy_drain_kernel(RankView rv, int ch, int64_t upto) {
  if (threadIdx.x == 0) drain_and_wait(rv, ch, upto);
}

// Test producer: n WRITEs on channel ch (block i: src_off + i*bytes -> dst_off + i*bytes
// at dst), then Drain(first + upto) where first is the index of the first WRITE;
// once it completes, result[i] = 1 if block i's first and last 16 bytes already
// match at the destination (only i <= upto is guaranteed), and
// result[n] = ns from the last push to the drain's completion.
__global__ void drain_test_kernel(RankView rv, int ch, int dst, int n, int64_t src_off, int64_t dst_off, int64_t bytes,
                                  int64_t upto, int32_t* result) {
  if (threadIdx.x != 0) return;
  int64_t first = -1;
  for (int i = 0; i < n; ++i) {
    uint64_t lo, hi;
    cmd_pack_dev(EPB_CMD_WRITE, (uint64_t)dst, (uint64_t)ch, (uint64_t)(src_off + i * bytes),
                 (uint64_t)(dst_off + i * bytes), (uint64_t)bytes, 0, lo, hi);
    const int64_t idx = fifo_push(rv, ch, lo, hi);
    if (idx < 0) return;
    if (i == 0) first = idx;
  }
  const uint64_t t0 = globaltimer();
  if (!drain_and_wait(rv, ch, upto < 0 ? -1 : first + upto)) return;
  const uint64_t t1 = globaltimer();
  const char* sp = rv.base + kRegionHeader + src_off;
  const char* dp = rv.peer[dst] + kRegionHeader + dst_off;
  const int64_t data = (int64_t)rv.region_bytes - (int64_t)kRegionHeader;
  const bool in_bounds = src_off + n * bytes <= data && dst_off + n * bytes <= data;
  for (int i = 0; i < n; ++i) {
    if (!in_bounds) {  // the proxy rejected these WRITEs (FaultError): nothing to compare
      result[i] = 0;
      continue;
    }
    const int4* a0 = reinterpret_cast<const int4*>(sp + i * bytes);
    const int4* b0 = reinterpret_cast<const int4*>(dp + i * bytes);
    const int64_t last = bytes / 16 - 1;
    const int4 x0 = __ldcv(a0), y0 = __ldcv(b0), x1 = __ldcv(a0 + last), y1 = __ldcv(b0 + last);
    result[i] = x0.x == y0.x && x0.y == y0.y && x0.z == y0.z && x0.w == y0.w && x1.x == y1.x && x1.y == y1.y &&
                x1.z == y1.z && x1.w == y1.w;
  }
  result[n] = (int32_t)min((uint64_t)INT32_MAX, t1 - t0);
}
}  // namespace epb

extern "C" int epb_proxy_drain(epb_t* ctx, int channel, int64_t upto, void* stream) {
  if (!ctx) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
  if (channel < 0 || channel >= ctx->cfg.fifo_channels) return epb_set_error(EPB_ERR_CONFIG, "no such FIFO channel");
  if (!ctx->proxy) return epb_set_error(EPB_ERR_UNSUPPORTED, "proxy not running");
  epb::proxy_drain_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(ctx->view(), channel, upto);
  EPB_CUDA(cudaGetLastError());
  return EPB_OK;
}

extern "C" int epb_debug_drain_test(epb_t* ctx, int channel, int dst, int n, int64_t src_off, int64_t dst_off,
                                    int64_t bytes, int64_t upto, int32_t* result, void* stream) {
  if (!ctx || !result) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  if (channel < 0 || channel >= ctx->cfg.fifo_channels || !ctx->proxy)
    return epb_set_error(EPB_ERR_CONFIG, "no such FIFO channel / proxy not running");
  if (dst < 0 || dst >= ctx->world || bytes < 16 || bytes % 16) return epb_set_error(EPB_ERR_CONFIG, "bad drain test");
  epb::drain_test_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(ctx->view(), channel, dst, n, src_off,
                                                                          dst_off, bytes, upto, result);
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

namespace epb {
__global__ void stamp_kernel(int64_t* dst) { *dst = (int64_t)globaltimer(); }

// Clock calibration: thread 0 stores %globaltimer into a pinned host word in a
// loop until the host raises *stop (or ~50 ms pass).
__global__ void clock_beacon_kernel(volatile int64_t* word, volatile int* stop) {
  const uint64_t t0 = globaltimer();
  while (!*stop) {
    const uint64_t t = globaltimer();
    *word = (int64_t)t;
    __threadfence_system();
    if (t - t0 > 50000000ull) break;
  }
}
}  // namespace epb

// Offset between %globaltimer (GPU, ns) and the host's CLOCK_REALTIME (ns):
// gpu_ns - host_ns, from the sample with the tightest host bracket around a
// read of the beacon word; *error_ns = half that bracket (plus the PCIe write
// latency of the beacon, not measured).  Used to put the proxy's host events
// and the kernels' %globaltimer marks on one time line (tools/trace_ll_proxy.py).
extern "C" int epb_clock_calibrate(int64_t* offset_ns, int64_t* error_ns) {
  if (!offset_ns) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  int64_t* word = nullptr;
  int* stop = nullptr;
  EPB_CUDA(cudaHostAlloc((void**)&word, sizeof(int64_t), cudaHostAllocMapped));
  EPB_CUDA(cudaHostAlloc((void**)&stop, sizeof(int), cudaHostAllocMapped));
  *word = 0;
  *stop = 0;
  int64_t *dword = nullptr;
  int* dstop = nullptr;
  cudaHostGetDevicePointer((void**)&dword, word, 0);
  cudaHostGetDevicePointer((void**)&dstop, stop, 0);
  cudaStream_t st;
  EPB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  epb::clock_beacon_kernel<<<1, 1, 0, st>>>(dword, dstop);
  auto now = []() {
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    return (int64_t)ts.tv_sec * 1000000000ll + ts.tv_nsec;
  };
  const int64_t deadline = now() + 20000000;
  while (*(volatile int64_t*)word == 0 && now() < deadline) {
  }
  int64_t best = INT64_MAX, off = 0;
  for (int i = 0; i < 20000; ++i) {
    const int64_t h0 = now();
    const int64_t g = *(volatile int64_t*)word;
    const int64_t h1 = now();
    if (g != 0 && h1 - h0 < best) {
      best = h1 - h0;
      off = g - (h0 + h1) / 2;
    }
  }
  *(volatile int*)stop = 1;
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  cudaFreeHost(word);
  cudaFreeHost(stop);
  if (best == INT64_MAX) return epb_set_error(EPB_ERR_CUDA, "clock beacon never ran");
  *offset_ns = off;
  if (error_ns) *error_ns = best / 2;
  return EPB_OK;
}

extern "C" int64_t epb_debug_ht_sig_offset(void) { return (int64_t)offsetof(epb::Meta, ht_sig); }

// Diagnostics: the LL proxy transport's device-side state, 16 int64:
// llp_self[2], ll_pcnt[2], ll_epoch[2], llp_grp[0][0][0..4], llp_grp[1][0][0..4]
extern "C" int epb_debug_ll_state(epb_t* ctx, int64_t* out16) {
  if (!ctx || !out16) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  epb::Scratch sc;
  EPB_CUDA(cudaMemcpy(&sc, epb::scratch_of(ctx->base), sizeof(sc), cudaMemcpyDeviceToHost));
  const int64_t v[16] = {sc.llp_self[0], sc.llp_self[1], sc.ll_pcnt[0], sc.ll_pcnt[1], sc.ll_epoch[0], sc.ll_epoch[1],
                         sc.llp_grp[0][0][0], sc.llp_grp[0][0][1], sc.llp_grp[0][0][2], sc.llp_grp[0][0][3],
                         sc.llp_grp[0][0][4], sc.llp_grp[1][0][0], sc.llp_grp[1][0][1], sc.llp_grp[1][0][2],
                         sc.llp_grp[1][0][3], sc.llp_grp[1][0][4]};
  std::memcpy(out16, v, sizeof(v));
  return EPB_OK;
}

extern "C" int epb_debug_stamp(int64_t* dst, void* stream) {
  epb::stamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(dst);
  EPB_CUDA(cudaGetLastError());
  return EPB_OK;
}

cudaError_t epb_pcopy_launch(const epb_pcopy_batch& b, cudaStream_t st) {
  if (b.njobs == 0) return cudaSuccess;
  epb::pcopy_kernel<<<b.nblocks, 512, 0, st>>>(b);
  return cudaGetLastError();
}

// Load this file's kernels now (see epb_preload_kernels, api.cpp).
cudaError_t epb_preload_fifo() {
  cudaFuncAttributes attr;
  for (const void* fn : {(const void*)epb::pcopy_kernel, (const void*)fifo_bench_kernel, (const void*)proxy_barrier_kernel, (const void*)epb::proxy_drain_kernel, (const void*)epb::drain_test_kernel, (const void*)epb::stamp_kernel, (const void*)epb::clock_beacon_kernel})
    if (cudaError_t e = cudaFuncGetAttributes(&attr, fn)) return e;
  return cudaSuccess;
}
