// api.cpp — context lifecycle, CUDA-IPC bootstrap and error plumbing of the
// C ABI (include/epb.h).  Replaces the reference's symmetric-region handshake
// ("exchanges the base address during handshake",
// PAPER.md:326-327) with CUDA IPC handles: each rank cudaMalloc's one region,
// exports its handle, and maps every peer's region into its address space so
// kernels can store straight into peer memory over NVLink.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unistd.h>
#include <string>

#include "ctx.h"

static thread_local std::string g_last_error;

int epb_set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int epb_cuda_check(cudaError_t e, const char* what) {
  return epb_set_error(EPB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

extern "C" const char* epb_last_error(void) { return g_last_error.c_str(); }

cudaError_t epb_launch_grid_sync(const void* func, dim3 grid, dim3 block, void** args, size_t smem,
                                 cudaStream_t st) {
  static const bool coop = [] {
    const char* s = std::getenv("EPB_COOP");
    return !(s && s[0] == '0');
  }();
  if (coop) return cudaLaunchCooperativeKernel(func, grid, block, args, smem, st);
  return cudaLaunchKernel(func, grid, block, args, smem, st);
}

// Per-call launch-config queries are a few microseconds each; the dispatch and
// combine calls sit on the host's critical path, so their answers are cached.
namespace {
std::mutex g_cfg_mu;
struct OccKey {
  const void* f;
  int threads;
  size_t smem;
  int dev;
};
std::vector<std::pair<OccKey, int>> g_occ;
std::vector<std::tuple<const void*, int, size_t>> g_smem;  // (func, device, granted max dynamic smem)
}  // namespace

int epb_max_active_blocks(const void* func, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(g_cfg_mu);
  for (auto& kv : g_occ)
    if (kv.first.f == func && kv.first.threads == threads && kv.first.smem == smem && kv.first.dev == dev)
      return kv.second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, func, threads, smem) != cudaSuccess) n = 0;
  g_occ.push_back({OccKey{func, threads, smem, dev}, n});
  return n;
}

// Raises the kernel's dynamic shared-memory limit to `smem` (static shared
// memory counts against the default 48 KB, so any nonzero request may need it).
// Shared-memory carveout for the path's kernels (EPB_CARVEOUT, percent,
// default 100 = maximum shared; negative = the driver's per-kernel choice).
// Set for the dispatch, layout and LL kernels; see dispatch_launch.
void epb_set_carveout(const void* func, bool enable) {
  static const int pct = [] {
    const char* s = std::getenv("EPB_CARVEOUT");
    return s ? std::atoi(s) : 100;
  }();
  const int want = enable ? pct : -1;  // -1 = cudaSharedmemCarveoutDefault
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> g(g_cfg_mu);
  for (auto& d : done)
    if (d.first == func) {
      if (d.second == want) return;
      d.second = want;
      cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, want);
      cudaGetLastError();
      return;
    }
  if (want < 0) {  // never changed: already the driver's choice
    done.emplace_back(func, want);
    return;
  }
  cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, want);
  cudaGetLastError();
  done.emplace_back(func, want);
}

bool epb_carveout_skip(const char* name) {
  const char* s = std::getenv("EPB_CARVEOUT_SKIP");  // e.g. "dispatch,combine" (measurement only)
  return s && std::strstr(s, name);
}

cudaError_t epb_ensure_smem(const void* func, size_t smem) {
  if (smem == 0) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(g_cfg_mu);
  for (auto& t : g_smem)
    if (std::get<0>(t) == func && std::get<1>(t) == dev && std::get<2>(t) >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) g_smem.emplace_back(func, dev, smem);
  return e;
}

extern "C" int epb_num_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

int epb_fifo_init(epb_ctx* ctx);     // proxy.cpp
void epb_fifo_free(epb_ctx* ctx);    // proxy.cpp

// Load every kernel of the library into the current device's context up front.
// With lazy module loading (the CUDA 12 default) a kernel is loaded at its first
// launch, and that load can wait for the device: an LL call whose dispatch is
// already spinning on proxy copies while the host issues the first combine
// launch stalls the proxy threads' copies behind the load (observed: every
// first LL proxy call of a fresh 4-GPU job timed out).
static cudaError_t epb_preload_kernels(int device) {
  static std::mutex m;
  static bool done[64] = {};
  std::lock_guard<std::mutex> g(m);
  if (device < 0 || device >= 64 || done[device]) return cudaSuccess;
  for (auto fn : {epb_preload_ll, epb_preload_combine, epb_preload_dispatch, epb_preload_layout, epb_preload_chunked,
                  epb_preload_fifo})
    if (cudaError_t e = fn()) return e;
  done[device] = true;
  return cudaSuccess;
}

extern "C" int epb_create(epb_t** out, int rank, int world, const epb_config_t* cfg) {
  if (!out || !cfg) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  *out = nullptr;
  if (world <= 0 || world > epb::kMaxRanks) return epb_set_error(EPB_ERR_CONFIG, "world size must be in [1, 8]");
  if (rank < 0 || rank >= world) return epb_set_error(EPB_ERR_CONFIG, "rank out of range");
  if (cfg->fifo_channels < 0 || cfg->fifo_channels > 64)
    return epb_set_error(EPB_ERR_CONFIG, "fifo_channels must be in [0, 64] (6-bit channel_id, command.py:37)");
  if (cfg->fifo_channels > 0 && (cfg->fifo_capacity <= 0 || (cfg->fifo_capacity & (cfg->fifo_capacity - 1))))
    return epb_set_error(EPB_ERR_CONFIG, "fifo_capacity must be a power of two (SPEC.md:108)");
  epb_ctx* ctx = new epb_ctx();
  ctx->rank = rank;
  ctx->world = world;
  ctx->cfg = *cfg;
  if (ctx->cfg.num_recv_slots <= 0) ctx->cfg.num_recv_slots = 2;
  if (const char* s = std::getenv("EPB_TIMEOUT_S")) ctx->timeout_ns = (uint64_t)(std::atof(s) * 1e9);
  if (const char* s = std::getenv("EPB_TRACE")) ctx->trace = std::atoi(s) != 0;
  if (const char* s = std::getenv("EPB_PROXY_CHMAP")) ctx->proxy_chmap = std::strcmp(s, "phase") == 0 ? 1 : 0;
  cudaError_t e = cudaGetDevice(&ctx->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (e == cudaSuccess) e = epb_preload_kernels(ctx->device);
  ctx->region_bytes = epb::kRegionHeader + epb::align_up(cfg->nvl_bytes, 4096) + epb::align_up(cfg->ll_bytes, 4096);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->base, ctx->region_bytes);
  if (e == cudaSuccess) e = cudaMemset(ctx->base, 0, ctx->region_bytes);
  if (e == cudaSuccess) e = cudaHostAlloc(&ctx->host, sizeof(epb::HostInfo), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    std::memset((void*)ctx->host, 0, sizeof(epb::HostInfo));
    e = cudaHostGetDevicePointer((void**)&ctx->host_dev, (void*)ctx->host, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    int rc = epb_cuda_check(e, "epb_create");
    if (ctx->base) cudaFree(ctx->base);
    if (ctx->host) cudaFreeHost((void*)ctx->host);
    delete ctx;
    return rc;
  }
  ctx->peer[rank] = ctx->base;
  if (int rc = epb_fifo_init(ctx)) {
    cudaFree(ctx->base);
    cudaFreeHost((void*)ctx->host);
    delete ctx;
    return rc;
  }
  *out = ctx;
  return EPB_OK;
}

extern "C" int epb_proxy_stop(epb_t* ctx);

extern "C" int epb_destroy(epb_t* ctx) {
  if (!ctx) return EPB_OK;
  cudaDeviceSynchronize();
  epb_proxy_stop(ctx);
  epb_fifo_free(ctx);
  if (ctx->barrier) epb_barrier_close(ctx->barrier, 1);
  for (int r = 0; r < ctx->world; ++r)
    if (ctx->peer_ipc[r] && ctx->peer[r]) cudaIpcCloseMemHandle(ctx->peer[r]);
  if (ctx->base) cudaFree(ctx->base);
  if (ctx->host) cudaFreeHost((void*)ctx->host);
  delete ctx;
  return EPB_OK;
}

extern "C" int epb_ipc_handle(epb_t* ctx, void* out_handle) {
  if (!ctx || !out_handle) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == EPB_IPC_HANDLE_BYTES, "ipc handle size");
  cudaIpcMemHandle_t h;
  EPB_CUDA(cudaIpcGetMemHandle(&h, ctx->base));
  std::memcpy(out_handle, &h, sizeof(h));
  return EPB_OK;
}

extern "C" int epb_open_peers(epb_t* ctx, const void* handles) {
  if (!ctx || !handles) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  const char* hb = static_cast<const char*>(handles);
  for (int r = 0; r < ctx->world; ++r) {
    if (r == ctx->rank || ctx->peer[r]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + (size_t)r * EPB_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return epb_set_error(EPB_ERR_CONNECTION, std::string("cudaIpcOpenMemHandle(rank ") +
                                                                         std::to_string(r) + "): " +
                                                                         cudaGetErrorString(e));
    ctx->peer[r] = static_cast<char*>(p);
    ctx->peer_ipc[r] = true;
    // touch the mapping with a copy now (read and write): the first copy-engine
    // access to a lazily enabled peer mapping can stall for ~100 ms, which must
    // not happen while a kernel spins on a proxy copy's completion
    const size_t probe = offsetof(epb::Scratch, trace) + epb::kMetaBytes;  // scratch words nobody reads remotely
    e = cudaMemcpy(ctx->base + probe, ctx->peer[r] + probe, 16, cudaMemcpyDefault);
    if (e == cudaSuccess) e = cudaMemcpy(ctx->peer[r] + probe + 16, ctx->base + probe + 16, 16, cudaMemcpyDefault);
    if (e != cudaSuccess) return epb_cuda_check(e, "peer mapping warm-up copy");
    // ... and every 2 MB page of the data region (read, then write back the
    // same bytes; nothing runs on the peer's region yet), so no copy engine
    // meets an untouched page of the mapping while a kernel waits on it
    const size_t stride = (size_t)2 << 20, start = epb::kRegionHeader;
    const size_t rows = ctx->region_bytes > start ? (ctx->region_bytes - start) / stride : 0;
    if (rows > 0) {
      void* tmp = nullptr;
      e = cudaMalloc(&tmp, rows * 16);
      if (e == cudaSuccess) e = cudaMemcpy2D(tmp, 16, ctx->peer[r] + start, stride, 16, rows, cudaMemcpyDefault);
      if (e == cudaSuccess) e = cudaMemcpy2D(ctx->peer[r] + start, stride, tmp, 16, 16, rows, cudaMemcpyDefault);
      if (tmp) cudaFree(tmp);
      if (e != cudaSuccess) return epb_cuda_check(e, "peer mapping page warm-up");
    }
  }
  if (!ctx->barrier) {  // the proxies' all-peer barrier segment, named after the job's handles
    const std::string name = epb_barrier_name(handles, (size_t)ctx->world * EPB_IPC_HANDLE_BYTES);
    if (int rc = epb_barrier_open(name.c_str(), ctx->world, ctx->rank, &ctx->barrier)) return rc;
  }
  return EPB_OK;
}

extern "C" int epb_link_local(epb_t* const* ctxs, int n) {
  if (!ctxs || n <= 0 || n > epb::kMaxLocal) return epb_set_error(EPB_ERR_PROTOCOL, "bad local group");
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i] || ctxs[i]->world != n || ctxs[i]->rank != i)
      return epb_set_error(EPB_ERR_CONFIG, "local group must hold ranks 0..n-1 of a world of n");
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) ctxs[i]->peer[j] = ctxs[j]->base;
  const struct {
    long pid;
    const void* first;
  } key{(long)getpid(), ctxs[0]};
  const std::string name = epb_barrier_name(&key, sizeof(key));
  for (int i = 0; i < n; ++i)
    if (!ctxs[i]->barrier)
      if (int rc = epb_barrier_open(name.c_str(), n, i, &ctxs[i]->barrier)) return rc;
  return EPB_OK;
}

extern "C" int epb_device_error(epb_t* ctx, int64_t* detail) {
  if (!ctx) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
  if (detail) *detail = ctx->host->err_detail;
  return (int)ctx->host->err_code;
}

extern "C" int epb_clear_device_error(epb_t* ctx) {
  if (!ctx) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
  ctx->host->err_code = 0;
  ctx->host->err_detail = 0;
  return EPB_OK;
}

extern "C" int epb_region(epb_t* ctx, void** base, size_t* bytes) {
  if (!ctx) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
  if (base) *base = ctx->base;
  if (bytes) *bytes = ctx->region_bytes;
  return EPB_OK;
}

extern "C" int64_t epb_arena_offset(void) { return (int64_t)epb::kRegionHeader; }

extern "C" int epb_trace(epb_t* ctx, int64_t* out64) {
  if (!ctx || !out64) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  EPB_CUDA(cudaMemcpy(out64, epb::scratch_of(ctx->base)->trace, sizeof(int64_t) * 64, cudaMemcpyDeviceToHost));
  return EPB_OK;
}
