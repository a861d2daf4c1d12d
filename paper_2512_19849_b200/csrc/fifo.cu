// fifo.cu — device-side FIFO microbenchmark (SPEC.md:513-521 fifo_stress with
// a GPU producer): one producer warp per channel pushes WRITE commands in
// batches of 32 slots (one 512-B burst over PCIe/C2C, one tail publish), then
// waits until the proxy reports them completed (check_completion).
#include <cuda_runtime.h>

#include <cstddef>

#include "ctx.h"
#include "ll_common.cuh"

namespace epb {

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
}  // namespace epb

extern "C" int64_t epb_debug_ht_sig_offset(void) { return (int64_t)offsetof(epb::Meta, ht_sig); }

extern "C" int epb_debug_stamp(int64_t* dst, void* stream) {
  epb::stamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(dst);
  return epb_cuda_check(cudaGetLastError(), "stamp");
}
