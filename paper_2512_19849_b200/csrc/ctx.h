// ctx.h — host-side state of one EP rank (the object behind epb_t*).
#pragma once

#include <atomic>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

struct epb_proxy;  // proxy.cpp

struct epb_ctx {
  int rank = 0, world = 1, device = 0;
  epb_config_t cfg{};
  size_t region_bytes = 0;
  char* base = nullptr;                 // cudaMalloc'd symmetric region
  char* peer[epb::kMaxRanks] = {};      // mapped peer regions (peer[rank] == base)
  bool peer_ipc[epb::kMaxRanks] = {};   // opened with cudaIpcOpenMemHandle
  epb::HostInfo* host = nullptr;        // pinned host view
  epb::HostInfo* host_dev = nullptr;    // device alias
  uint32_t host_seq = 0;                // normal dispatch calls so far: the tag of the host count words
  uint64_t ht_disp_calls = 0, ht_comb_calls = 0;  // proxy transport calls so far (ht_sig targets)
  uint64_t ll_proxy_disp = 0, ll_proxy_comb = 0;  // proxy-transport LL calls so far (signal targets)
  int num_sms = 148;
  int proxy_chmap = 0;                  // proxy_thread_of mode (EPB_PROXY_CHMAP=phase -> 1)
  uint64_t timeout_ns = 30ull * 1000 * 1000 * 1000;
  int trace = 0;                        // EPB_TRACE=1: kernels record phase timestamps
  int ll_grid[2] = {0, 0};              // LL dispatch / combine grid width, pinned at the first call
  // LL bookkeeping of the last dispatch (shape) for combine validation.
  int ll_last_tokens = -1;
  // GPU -> CPU command FIFOs (pinned, mapped) and the proxy.
  std::vector<int64_t*> fifo_host;      // ctl arrays (kernels.py:23-31 layout)
  std::vector<int64_t*> fifo_dev;       // device aliases
  epb_proxy* proxy = nullptr;
  std::vector<int64_t> proxy_trace;     // the last stopped proxy's trace events (4 int64 each)
  epb_barrier_t* barrier = nullptr;     // proxy all-peer barrier (barrier.cpp)

  size_t arena_off() const { return epb::kRegionHeader; }
  size_t ll_off() const { return epb::kRegionHeader + epb::align_up(cfg.nvl_bytes, 4096); }

  epb::RankView view() const {
    epb::RankView v{};
    v.rank = rank;
    v.world = world;
    v.base = base;
    for (int i = 0; i < epb::kMaxRanks; ++i) v.peer[i] = peer[i];
    v.host = host_dev;
    v.timeout_ns = timeout_ns;
    v.trace = trace;
    v.region_bytes = region_bytes;
    return v;
  }
};

// Launch a kernel whose blocks wait on each other.  Default: a cooperative
// launch (co-residency guaranteed by the driver).  EPB_COOP=0 switches to a
// plain launch (grid is still sized to fit one wave); api.cpp.
cudaError_t epb_launch_grid_sync(const void* func, dim3 grid, dim3 block, void** args, size_t smem,
                                 cudaStream_t st);

// Cached launch-configuration queries (api.cpp).
int epb_max_active_blocks(const void* func, int threads, size_t smem);
cudaError_t epb_ensure_smem(const void* func, size_t smem);
void epb_set_carveout(const void* func, bool enable = true);
bool epb_carveout_skip(const char* name);

// SM copy engine of the CPU proxy (EPB_PROXY_ENGINE=sm; fifo.cu): the proxy
// thread launches one copy kernel per sweep instead of copy-engine copies.  A
// job = contiguous segments to one destination, then an optional stream-ordered
// 8-byte signal (the piggybacked count / ATOMIC value), written by the job's
// last block after every block's copies.
struct epb_pcopy_seg {
  const char* src;
  char* dst;
  uint64_t len;
};
struct epb_pcopy_job {
  int dest, seg0, nseg, blocks, block0;
  uint64_t* sig;      // nullptr: no signal
  uint64_t sig_val;
};
constexpr int kPcopyJobs = 8, kPcopySegs = 16;  // small launch parameters (~0.7 KB)
struct epb_pcopy_batch {
  int njobs, nsegs, nblocks;
  uint32_t* tickets;  // [kPcopyJobs] device counters, zero between launches
  int64_t* stamp;     // tracing: [4] = %globaltimer at kernel start, last signal, last block start,
                      // last block's copies done (or nullptr)
  epb_pcopy_job jobs[kPcopyJobs];
  epb_pcopy_seg segs[kPcopySegs];
};
cudaError_t epb_pcopy_launch(const epb_pcopy_batch& b, cudaStream_t st);

// Per-file kernel preloads (each .cu), run once per device by epb_create.
cudaError_t epb_preload_ll();
cudaError_t epb_preload_combine();
cudaError_t epb_preload_dispatch();
cudaError_t epb_preload_layout();
cudaError_t epb_preload_chunked();
cudaError_t epb_preload_fifo();

// proxy threads a context runs (proxy.cpp): channel c is served by thread c % n
int epb_proxy_nthreads(const epb_ctx* ctx);

// name of the job-wide barrier segment (barrier.cpp)
std::string epb_barrier_name(const void* bytes, size_t n);

// normal-mode arena geometry and group validation (layout.cu)
int compute_recv_layout(const epb_ctx* ctx, int hidden, int k, epb_recv_layout_t* L);
int check_group(epb_t* const* ctxs, int n);

// error plumbing (api.cpp)
int epb_set_error(int code, const std::string& msg);
int epb_cuda_check(cudaError_t e, const char* what);
#define EPB_CUDA(call)                                              \
  do {                                                              \
    cudaError_t _e = (call);                                        \
    if (_e != cudaSuccess) return epb_cuda_check(_e, #call);        \
  } while (0)
