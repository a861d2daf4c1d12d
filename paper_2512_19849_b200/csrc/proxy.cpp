// proxy.cpp — GPU -> CPU command FIFOs and the multithreaded CPU proxy.
//
// FIFO: one pinned, device-mapped control
// array per channel in the reference layout (kernels.py:23-31).  The device
// producer (ll.cu fifo_push) writes 16-byte TransferCmds (command.py:8-13) and
// publishes TAIL with st.release.sys; the proxy reads TAIL with an acquire
// load, consumes the slots, publishes HEAD, and publishes COMPLETED (= number
// of commands whose effects have finished) once the copies it issued are done.
//
// Proxy: proxy_threads OS threads per
// rank; thread i owns channels {c : c % threads == i} and never shares mutable
// state with another thread.  Each thread issues on its own
// CUDA stream, so commands of one channel take effect in FIFO order (channels
// of one thread are additionally ordered among themselves, which "cross-FIFO
// ordering is not guaranteed" permits).
//   WRITE   -> offset translation (the symmetric data region — normal arena, then
//              the LL region — starting after the Meta/Scratch header;
//              SPEC.md:237-241) and a
//              cudaMemcpyAsync; contiguous WRITEs to the same peer coalesce
//              into one copy; FLAG_PIGGYBACK_ATOMIC then bumps the receiver's
//              proxy_sig[channel][me] counter on the same stream (ordered after
//              the data: the LL completion fence of PAPER.md:343-346).
//   ATOMIC  -> counter += value at dst_offset of the peer region, stream-ordered
//              after all earlier commands of the channel.  The peer counter has
//              a single writer (this channel), so the add is a shadow-value store.
//   DRAIN   -> waits for every copy issued on the channel.
//   BARRIER -> drains the channel, then the all-peer rendezvous of barrier.cpp
//              (SPEC.md:274-282); SameRail completes at once on one node.
//              The thread blocks meanwhile ("Barrier and Drain are blocking").
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstring>
#include <deque>
#include <thread>
#include <unordered_map>
#include <vector>

#include "ctx.h"

struct epb_proxy {
  epb_ctx* ctx = nullptr;
  std::vector<std::thread> threads;
  std::atomic<bool> stop{false};
  std::atomic<bool> count_only{false};
  std::atomic<int64_t> served{0}, copies{0}, atomics{0};
};

namespace {

inline int64_t load_acquire(const int64_t* p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }
inline void store_release(int64_t* p, int64_t v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }

constexpr int kValueRing = 4096;

struct PendingCopy {
  int dst = -1;
  char* src = nullptr;
  char* dstp = nullptr;
  size_t len = 0;
};

struct ChanState {
  int ch = 0;
  cudaStream_t st = nullptr;
  int64_t head = 0;
  std::deque<std::pair<cudaEvent_t, int64_t>> inflight;
  std::vector<cudaEvent_t> pool;
  uint64_t* vals = nullptr;  // pinned value ring for counter stores
  int64_t vi = 0;
  PendingCopy pend;
};

void proxy_error(epb_ctx* ctx, int code, int64_t detail) {
  ctx->host->err_detail = detail;
  ctx->host->err_code = code;
}

void flush(epb_proxy* px, ChanState& cs) {
  if (cs.pend.len == 0) return;
  cudaMemcpyAsync(cs.pend.dstp, cs.pend.src, cs.pend.len, cudaMemcpyDefault, cs.st);
  px->copies.fetch_add(1, std::memory_order_relaxed);
  cs.pend = PendingCopy{};
}

void signal(epb_proxy* px, ChanState& cs, std::unordered_map<uint64_t, uint64_t>& shadow, int dst, uint64_t off,
            uint64_t v) {
  epb_ctx* ctx = px->ctx;
  const uint64_t key = ((uint64_t)dst << 40) | off;
  const uint64_t nv = (shadow[key] += v);
  uint64_t* slot = &cs.vals[cs.vi++ % kValueRing];
  *slot = nv;
  cudaMemcpyAsync(ctx->peer[dst] + off, slot, sizeof(uint64_t), cudaMemcpyDefault, cs.st);
  px->atomics.fetch_add(1, std::memory_order_relaxed);
}

void serve(epb_proxy* px, ChanState& cs, std::unordered_map<uint64_t, uint64_t>& shadow, uint64_t lo, uint64_t hi) {
  epb_ctx* ctx = px->ctx;
  px->served.fetch_add(1, std::memory_order_relaxed);
  if (hi >> 54) {  // reserved bits (command.py:87-88)
    proxy_error(ctx, EPB_ERR_PROTOCOL, (int64_t)(hi >> 54));
    return;
  }
  if (px->count_only.load(std::memory_order_relaxed)) return;
  const int kind = (int)(lo & 3);
  const int dst = (int)((lo >> 2) & 0xFFF);
  const int ch_id = (int)((lo >> 14) & 0x3F);
  const uint64_t so = (lo >> 20) & 0xFFFFFFFFull;
  const uint64_t dof = ((lo >> 52) | ((hi & 0xFFFFFull) << 12)) & 0xFFFFFFFFull;
  const uint64_t len = (hi >> 20) & 0xFFFFFFFFull;
  const int flags = (int)((hi >> 52) & 3);
  if (dst >= ctx->world || ctx->peer[dst] == nullptr) {
    proxy_error(ctx, EPB_ERR_CONNECTION, dst);
    return;
  }
  switch (kind) {
    case EPB_CMD_WRITE: {
      // offsets are relative to the arena start (normal arena, then the LL region)
      const size_t data = ctx->ll_off() - epb::kRegionHeader + ctx->cfg.ll_bytes;
      if (so + len > data || dof + len > data) {  // FaultError(rank, offset, length), errors.py:20-27
        proxy_error(ctx, EPB_ERR_FAULT, (int64_t)((uint64_t)dst << 56 | (so + len > data ? so : dof)));
        return;
      }
      char* s = ctx->base + epb::kRegionHeader + so;
      char* d = ctx->peer[dst] + epb::kRegionHeader + dof;
      PendingCopy& p = cs.pend;
      if (p.len > 0 && p.dst == dst && p.src + p.len == s && p.dstp + p.len == d) {
        p.len += len;
      } else {
        flush(px, cs);
        if (len > 0) cs.pend = PendingCopy{dst, s, d, (size_t)len};
      }
      if (flags & EPB_FLAG_PIGGYBACK_ATOMIC) {
        flush(px, cs);
        signal(px, cs, shadow, dst, offsetof(epb::Meta, proxy_sig) + sizeof(uint64_t) * ((size_t)ch_id * epb::kMaxRanks + ctx->rank), 1);
      }
      break;
    }
    case EPB_CMD_ATOMIC: {
      flush(px, cs);
      if (dof % 8 != 0 || dof + 8 > epb::kMetaBytes) {
        proxy_error(ctx, EPB_ERR_FAULT, (int64_t)((uint64_t)dst << 56 | dof));
        return;
      }
      signal(px, cs, shadow, dst, dof, len);
      break;
    }
    case EPB_CMD_DRAIN:
      flush(px, cs);
      cudaStreamSynchronize(cs.st);
      break;
    case EPB_CMD_BARRIER: {
      // everything this channel issued before the barrier has landed, then
      // the all-peer rendezvous (barrier.cpp); COMPLETED advances after it
      flush(px, cs);
      cudaStreamSynchronize(cs.st);
      const double timeout_s = (double)ctx->timeout_ns * 1e-9;
      if (!ctx->barrier) proxy_error(ctx, EPB_ERR_CONNECTION, 0xba);
      else if (epb_barrier_wait(ctx->barrier, (flags & EPB_FLAG_SAME_RAIL_BARRIER) != 0, timeout_s) != EPB_OK)
        proxy_error(ctx, EPB_ERR_DEADLOCK, 0xbb);
      break;
    }
    default:
      flush(px, cs);
      proxy_error(ctx, EPB_ERR_UNSUPPORTED, kind);
      break;
  }
}

void proxy_main(epb_proxy* px, int tid, int nthreads) {
  epb_ctx* ctx = px->ctx;
  cudaSetDevice(ctx->device);
  const int C = ctx->cfg.fifo_channels;
  const int64_t cap = ctx->cfg.fifo_capacity, mask = cap - 1;
  std::vector<ChanState> chans;
  // one stream per proxy thread: the thread's channels then execute in the
  // order it serves them (stronger than required), and a rank needs only
  // proxy_threads hardware queues — CUDA multiplexes streams onto
  // CUDA_DEVICE_MAX_CONNECTIONS queues, and a proxy copy that lands in the
  // queue of a kernel spinning on that very copy would wait for it forever
  cudaStream_t st = nullptr;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int ch = tid; ch < C; ch += nthreads) {
    ChanState cs;
    cs.ch = ch;
    cs.st = st;
    cudaHostAlloc(&cs.vals, sizeof(uint64_t) * kValueRing, cudaHostAllocDefault);
    cs.head = load_acquire(&ctx->fifo_host[ch][EPB_CTL_HEAD]);
    chans.push_back(cs);
  }
  std::unordered_map<uint64_t, uint64_t> shadow;
  int64_t idle = 0;
  while (!px->stop.load(std::memory_order_relaxed)) {
    bool any = false;
    for (ChanState& cs : chans) {
      int64_t* ctl = ctx->fifo_host[cs.ch];
      const int64_t tail = load_acquire(&ctl[EPB_CTL_TAIL]);
      if (tail != cs.head) {
        while (cs.head < tail) {
          const int64_t s = EPB_CTL_SLOT0 + 2 * (cs.head & mask);
          const uint64_t lo = (uint64_t)ctl[s], hi = (uint64_t)ctl[s + 1];
          ++cs.head;
          serve(px, cs, shadow, lo, hi);
        }
        flush(px, cs);
        store_release(&ctl[EPB_CTL_HEAD], cs.head);
        if (px->count_only.load(std::memory_order_relaxed)) {
          store_release(&ctl[EPB_CTL_COMPLETED], cs.head);
        } else {
          cudaEvent_t ev;
          if (cs.pool.empty()) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
          else {
            ev = cs.pool.back();
            cs.pool.pop_back();
          }
          cudaEventRecord(ev, cs.st);
          cs.inflight.emplace_back(ev, cs.head);
        }
        any = true;
      }
      while (!cs.inflight.empty() && cudaEventQuery(cs.inflight.front().first) == cudaSuccess) {
        store_release(&ctl[EPB_CTL_COMPLETED], cs.inflight.front().second);
        cs.pool.push_back(cs.inflight.front().first);
        cs.inflight.pop_front();
      }
      if (!cs.inflight.empty()) any = true;
    }
    if (any) {
      idle = 0;
    } else if (++idle < 200000) {
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    } else {
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  cudaStreamSynchronize(st);
  for (ChanState& cs : chans) {
    for (auto& pr : cs.inflight) cudaEventDestroy(pr.first);
    for (auto ev : cs.pool) cudaEventDestroy(ev);
    cudaFreeHost(cs.vals);
  }
  cudaStreamDestroy(st);
}

}  // namespace

int epb_fifo_init(epb_ctx* ctx) {
  const int C = ctx->cfg.fifo_channels;
  if (C == 0) return EPB_OK;
  const int64_t cap = ctx->cfg.fifo_capacity;
  const size_t bytes = sizeof(int64_t) * (EPB_CTL_SLOT0 + 2 * cap);
  for (int ch = 0; ch < C; ++ch) {
    int64_t* h = nullptr;
    int64_t* d = nullptr;
    EPB_CUDA(cudaHostAlloc((void**)&h, bytes, cudaHostAllocMapped));
    std::memset(h, 0, bytes);
    EPB_CUDA(cudaHostGetDevicePointer((void**)&d, h, 0));
    ctx->fifo_host.push_back(h);
    ctx->fifo_dev.push_back(d);
  }
  // producer-side state lives in device memory (Scratch)
  epb::Scratch* sc = epb::scratch_of(ctx->base);
  uint64_t table[epb::kMaxFifo] = {};
  for (int ch = 0; ch < C; ++ch) table[ch] = reinterpret_cast<uint64_t>(ctx->fifo_dev[ch]);
  int32_t cc[2] = {C, (int32_t)cap};
  EPB_CUDA(cudaMemcpy(sc->fifo_ctl, table, sizeof(table), cudaMemcpyHostToDevice));
  EPB_CUDA(cudaMemset(sc->fifo_tail, 0, sizeof(int64_t) * epb::kMaxFifo));
  EPB_CUDA(cudaMemset(sc->fifo_head, 0, sizeof(int64_t) * epb::kMaxFifo));
  EPB_CUDA(cudaMemcpy(&sc->fifo_channels, cc, sizeof(cc), cudaMemcpyHostToDevice));
  return EPB_OK;
}

void epb_fifo_free(epb_ctx* ctx) {
  for (int64_t* h : ctx->fifo_host) cudaFreeHost(h);
  ctx->fifo_host.clear();
  ctx->fifo_dev.clear();
}

int epb_proxy_set_count_only(epb_ctx* ctx, bool on) {
  if (ctx->proxy) ctx->proxy->count_only.store(on);
  return EPB_OK;
}

extern "C" int epb_fifo_ctl(epb_t* ctx, int channel, int64_t** host_ctl, int64_t* capacity) {
  if (!ctx || !host_ctl) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  if (channel < 0 || channel >= (int)ctx->fifo_host.size()) return epb_set_error(EPB_ERR_CONFIG, "no such FIFO channel");
  *host_ctl = ctx->fifo_host[channel];
  if (capacity) *capacity = ctx->cfg.fifo_capacity;
  return EPB_OK;
}

extern "C" int epb_proxy_start(epb_t* ctx) {
  if (!ctx) return epb_set_error(EPB_ERR_PROTOCOL, "null context");
  if (ctx->proxy) return EPB_OK;
  if (ctx->cfg.fifo_channels <= 0) return epb_set_error(EPB_ERR_CONFIG, "no FIFO channels configured");
  const int n = std::max(1, std::min(ctx->cfg.proxy_threads, ctx->cfg.fifo_channels));
  epb_proxy* px = new epb_proxy();
  px->ctx = ctx;
  for (int i = 0; i < n; ++i) px->threads.emplace_back(proxy_main, px, i, n);
  ctx->proxy = px;
  return EPB_OK;
}

extern "C" int epb_proxy_stop(epb_t* ctx) {
  if (!ctx || !ctx->proxy) return EPB_OK;
  ctx->proxy->stop.store(true);
  for (auto& t : ctx->proxy->threads) t.join();
  delete ctx->proxy;
  ctx->proxy = nullptr;
  return EPB_OK;
}

extern "C" int epb_proxy_stats(epb_t* ctx, int64_t* out3) {
  if (!ctx || !out3) return epb_set_error(EPB_ERR_PROTOCOL, "null argument");
  if (!ctx->proxy) {
    out3[0] = out3[1] = out3[2] = 0;
    return EPB_OK;
  }
  out3[0] = ctx->proxy->served.load();
  out3[1] = ctx->proxy->copies.load();
  out3[2] = ctx->proxy->atomics.load();
  return EPB_OK;
}
