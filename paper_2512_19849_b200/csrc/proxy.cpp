// proxy.cpp — GPU -> CPU command FIFOs and the multithreaded CPU proxy.
//
// FIFO: one pinned, device-mapped control
// array per channel in the reference layout (kernels.py:23-31).  The device
// producer (ll_common.cuh fifo_push) writes 16-byte TransferCmds
// (command.py:8-13) and publishes TAIL with st.release.sys; the proxy reads
// TAIL with an acquire load, consumes the slots, publishes HEAD, and publishes
// COMPLETED (a high-water mark, SPEC.md:80-89 mark_completed) once the copies
// it issued for them are done.
//
// Proxy: proxy_threads OS threads per
// rank; thread i owns channels {c : c % threads == i} and shares no mutable
// state with another thread.  Each thread issues on its own
// CUDA stream per destination rank, so commands to one destination take
// effect in the order the thread serves them.
//   WRITE   -> offset translation (the symmetric data region — normal arena,
//              then the LL region — starting after the Meta/Scratch header;
//              SPEC.md:237-241) and a cudaMemcpyAsync on the destination's
//              stream; contiguous WRITEs to the same peer served in one sweep
//              (from any of the thread's channels) coalesce into one copy.
//              FLAG_PIGGYBACK_ATOMIC: after the sweep's copies to that peer,
//              ONE stream-ordered cuStreamWriteValue64 publishes the thread's
//              cumulative count of piggybacked WRITEs to the peer's
//              proxy_sig[kind*32 + thread][me] (kind 0: channels of the first
//              half — LL dispatch; 1: second half — LL combine).  The value
//              store follows the copies on the same stream: the LL completion
//              fence of PAPER.md:343-346 without a host round trip.
//   ATOMIC  -> counter += value at dst_offset of the peer region, as a
//              stream-ordered cuStreamWriteValue64 of the cumulative value
//              (single writer per counter: the channel's thread).
//   DRAIN   -> length_or_value = Idx + 1 (0: everything): waits until every
//              copy issued for commands <= Idx of the channel has completed,
//              then marks the Drain completed.
//   BARRIER -> drains the thread's streams, then the all-peer rendezvous of
//              barrier.cpp; SameRail completes at once on
//              one node.  "Barrier and Drain are blocking".
// Every CUDA call is checked; a failure is reported through the host error
// word (EPB_ERR_CUDA, detail = the cudaError_t), which the waiting kernels and
// the host API surface as an exception.
// Tracing (EPB_TRACE=1): per-thread events {host ns, kind, a, b} for the phase
// trace of tools/trace_ll_proxy.py (read with epb_proxy_trace).
#include <cuda.h>
#include <cuda_runtime.h>
#include <time.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "ctx.h"
#include "pcopy_plan.h"

namespace {
struct TraceEv {
  int64_t t_ns, kind, a, b;
};
}  // namespace

struct epb_proxy {
  epb_ctx* ctx = nullptr;
  std::vector<std::thread> threads;
  std::atomic<bool> stop{false};
  std::atomic<int> ready{0};  // threads past their warm-up (epb_proxy_start waits for all)
  std::atomic<bool> count_only{false};
  std::atomic<int64_t> served{0}, copies{0}, atomics{0};
  std::mutex trace_m;
  std::vector<TraceEv> trace;  // the threads' events, handed over at thread exit
};

namespace {

inline int64_t load_acquire(const int64_t* p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }
inline void store_release(int64_t* p, int64_t v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }
inline void store_max_release(int64_t* p, int64_t v) {
  int64_t cur = __atomic_load_n(p, __ATOMIC_RELAXED);
  while (cur < v && !__atomic_compare_exchange_n(p, &cur, v, false, __ATOMIC_RELEASE, __ATOMIC_RELAXED)) {
  }
}
inline int64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return (int64_t)ts.tv_sec * 1000000000ll + ts.tv_nsec;
}

// cuStreamWriteValue64 through the runtime's driver entry point (no -lcuda).
using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
WriteValue64Fn write_value64() {
  static WriteValue64Fn fn = []() -> WriteValue64Fn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<WriteValue64Fn>(p);
  }();
  return fn;
}

struct PendingCopy {
  char* src = nullptr;
  char* dstp = nullptr;
  size_t len = 0;
};

struct DestState {              // one per destination rank this thread writes to
  cudaStream_t st = nullptr;
  PendingCopy pend;
  bool used = false;            // work issued in the current sweep
  uint64_t sig[2] = {0, 0};     // cumulative piggybacked WRITEs [LL dispatch | LL combine]
  bool sig_dirty[2] = {false, false};
};

struct ChanState {
  int ch = 0;
  int64_t head = 0;
  int64_t served_upto = 0;      // commands served (== head after a sweep)
};

struct Inflight {
  std::vector<cudaEvent_t> evs;
  std::vector<std::pair<int, int64_t>> marks;  // (channel, COMPLETED value) once evs are done
};

// SM copy engine (EPB_PROXY_ENGINE=sm): a destination's pending copies and up
// to two signals, turned into one job of the sweep's copy-kernel launch
struct Worker {
  epb_proxy* px;
  epb_ctx* ctx;
  int tid, nthreads, half;
  bool sm_engine = false;
  cudaStream_t kst = nullptr;     // SM engine: the thread's copy-kernel stream
  bool kst_used = false;
  uint32_t* tickets = nullptr;    // SM engine: per-job last-block tickets (device)
  int64_t* stamps = nullptr;      // SM engine + tracing: [kStampRing][2] device stamps per launch
  int64_t launches = 0;
  // SM engine: bytes per copy-kernel block (EPB_PCOPY_BLOCK_KB).  64 KB: LL pair 126 us
  // at EP=4; 32 / 16 / 8 KB: 137 / 140 / 140 us — the extra blocks cannot all sit
  // beside the LL kernel's and start in a second wave (profiles/r02_proxy_engine_n4.txt)
  int64_t pcopy_block = 65536;
  static constexpr int kStampRing = 512;
  std::vector<PJob> jobs;         // SM engine: the sweep's open jobs, in issue order
  std::vector<ChanState> chans;
  std::vector<DestState> dests;
  std::unordered_map<uint64_t, uint64_t> shadow;  // ATOMIC counters: (dst, off) -> cumulative value
  std::deque<Inflight> inflight;
  std::vector<cudaEvent_t> pool;
  std::vector<TraceEv> trace;
  bool tracing = false;

  void error(int code, int64_t detail) {
    ctx->host->err_detail = detail;
    ctx->host->err_code = code;
  }
  bool ok(cudaError_t e) {
    if (e == cudaSuccess) return true;
    error(EPB_ERR_CUDA, (int64_t)e);
    return false;
  }
  void tr(int64_t kind, int64_t a, int64_t b) {
    if (tracing && trace.size() < (1u << 20)) trace.push_back({now_ns(), kind, a, b});
  }
  DestState& dest(int d) {
    DestState& ds = dests[d];
    if (!ds.st) ok(cudaStreamCreateWithFlags(&ds.st, cudaStreamNonBlocking));
    return ds;
  }
  cudaEvent_t event() {
    cudaEvent_t ev = nullptr;
    if (!pool.empty()) {
      ev = pool.back();
      pool.pop_back();
    } else {
      ok(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    return ev;
  }

  // SM engine: the open job of destination d (a job that already carries a
  // signal takes no more copies: its signal must follow only its own copies)
  PJob& job_for(int d, bool for_copy) {
    for (int i = (int)jobs.size() - 1; i >= 0; --i)
      if (jobs[i].dest == d) {
        if ((for_copy && jobs[i].nsig > 0) || jobs[i].nsig == 2) break;
        return jobs[i];
      }
    if (jobs.size() >= (size_t)kPcopyJobs) launch_jobs();
    jobs.emplace_back();
    jobs.back().dest = d;
    return jobs.back();
  }
  // one copy-kernel launch for the open jobs (several if they exceed a batch)
  int64_t* next_stamp() {
    if (!stamps) return nullptr;
    int64_t* p = stamps + 4 * (launches % kStampRing);
    ++launches;
    return p;
  }
  void launch_jobs() {
    for (epb_pcopy_batch& b : pcopy_plan(jobs, pcopy_block)) {
      b.tickets = tickets;
      b.stamp = next_stamp();
      for (int j = 0; j < b.njobs; ++j)
        if (b.jobs[j].sig) tr(3, b.jobs[j].dest, (int64_t)b.jobs[j].sig_val);
      tr(6, -1, (int64_t)b.nblocks);
      ok(epb_pcopy_launch(b, kst));
      px->copies.fetch_add(1, std::memory_order_relaxed);
      tr(2, -1, 0);
    }
    jobs.clear();
    kst_used = true;
  }

  void flush(int d) {
    DestState& ds = dests[d];
    if (ds.pend.len == 0) return;
    if (sm_engine) {
      PJob& J = job_for(d, true);
      J.segs.push_back({ds.pend.src, ds.pend.dstp, (uint64_t)ds.pend.len});
      J.bytes += ds.pend.len;
      if (J.segs.size() >= (size_t)kPcopySegs / 2) launch_jobs();
      ds.pend = PendingCopy{};
      return;
    }
    tr(6, d, (int64_t)ds.pend.len);
    ok(cudaMemcpyAsync(ds.pend.dstp, ds.pend.src, ds.pend.len, cudaMemcpyDefault, ds.st));
    tr(2, d, (int64_t)ds.pend.len);
    px->copies.fetch_add(1, std::memory_order_relaxed);
    ds.pend = PendingCopy{};
    ds.used = true;
  }
  void write_value(int d, uint64_t off, uint64_t value) {
    if (sm_engine) {
      PJob& J = job_for(d, false);
      J.sig[J.nsig] = reinterpret_cast<uint64_t*>(ctx->peer[d] + off);
      J.val[J.nsig] = value;
      ++J.nsig;
      px->atomics.fetch_add(1, std::memory_order_relaxed);
      return;
    }
    DestState& ds = dest(d);
    WriteValue64Fn fn = write_value64();
    if (!fn) {
      error(EPB_ERR_CUDA, (int64_t)cudaErrorNotSupported);
      return;
    }
    // default flags: the write is preceded by a memory barrier on the stream,
    // so the copies issued before it are visible when the value is
    tr(7, d, (int64_t)value);
    CUresult r = fn(reinterpret_cast<CUstream>(ds.st), reinterpret_cast<CUdeviceptr>(ctx->peer[d] + off), value, 0);
    if (r != CUDA_SUCCESS) error(EPB_ERR_CUDA, 100000 + (int64_t)r);
    tr(3, d, (int64_t)value);
    px->atomics.fetch_add(1, std::memory_order_relaxed);
    ds.used = true;
  }
  // flush every destination's copy, then publish the piggyback signals
  void flush_all() {
    for (int d = 0; d < ctx->world; ++d) {
      flush(d);
      DestState& ds = dests[d];
      for (int k = 0; k < 2; ++k) {
        if (!ds.sig_dirty[k]) continue;
        ds.sig_dirty[k] = false;
        const size_t idx = (size_t)(k * 32 + tid) * epb::kMaxRanks + ctx->rank;
        write_value(d, offsetof(epb::Meta, proxy_sig) + sizeof(uint64_t) * idx, ds.sig[k]);
      }
    }
    if (sm_engine && !jobs.empty()) launch_jobs();
  }
  // events on every stream used since the last call (one completion point)
  std::vector<cudaEvent_t> mark_streams(bool all) {
    std::vector<cudaEvent_t> evs;
    if (sm_engine && (kst_used || all)) {
      cudaEvent_t ev = event();
      if (ok(cudaEventRecord(ev, kst))) evs.push_back(ev);
      kst_used = false;
    }
    for (int d = 0; d < ctx->world; ++d) {
      DestState& ds = dests[d];
      if (!ds.st || !(ds.used || all)) continue;
      cudaEvent_t ev = event();
      tr(8, d, 0);
      if (ok(cudaEventRecord(ev, ds.st))) evs.push_back(ev);
      tr(9, d, 0);
      ds.used = false;
    }
    return evs;
  }
  void wait_events(const std::vector<cudaEvent_t>& evs) {
    for (cudaEvent_t ev : evs) ok(cudaEventSynchronize(ev));
  }

  uint64_t seed_counter(int d, uint64_t off) {
    // first use of a counter in this proxy's life: continue from the value in
    // device memory (a restarted proxy must not publish smaller counts).  Read
    // on the destination's non-blocking stream: a legacy-stream copy would
    // wait for kernels that may be spinning on this very proxy.
    DestState& ds = dest(d);
    uint64_t v = 0;
    if (ok(cudaMemcpyAsync(&v, ctx->peer[d] + off, sizeof(v), cudaMemcpyDefault, ds.st))) ok(cudaStreamSynchronize(ds.st));
    return v;
  }

  void serve(ChanState& cs, int64_t idx, uint64_t lo, uint64_t hi, std::vector<cudaEvent_t>* cut, int64_t cut_at) {
    px->served.fetch_add(1, std::memory_order_relaxed);
    if (hi >> 54) {  // reserved bits (command.py:87-88)
      error(EPB_ERR_PROTOCOL, (int64_t)(hi >> 54));
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
    if (kind == EPB_CMD_WRITE || kind == EPB_CMD_ATOMIC) {
      if (dst >= ctx->world || ctx->peer[dst] == nullptr) {
        error(EPB_ERR_CONNECTION, dst);
        return;
      }
    }
    switch (kind) {
      case EPB_CMD_WRITE: {
        // offsets are relative to the arena start (normal arena, then the LL region)
        const size_t data = ctx->ll_off() - epb::kRegionHeader + ctx->cfg.ll_bytes;
        if (so + len > data || dof + len > data) {  // FaultError(rank, offset, length), errors.py:20-27
          error(EPB_ERR_FAULT, (int64_t)((uint64_t)dst << 56 | (so + len > data ? so : dof)));
          return;
        }
        char* s = ctx->base + epb::kRegionHeader + so;
        char* d = ctx->peer[dst] + epb::kRegionHeader + dof;
        DestState& ds = dest(dst);
        PendingCopy& p = ds.pend;
        if (p.len > 0 && p.src + p.len == s && p.dstp + p.len == d) {
          p.len += len;
        } else if (len > 0) {
          flush(dst);
          ds.pend = PendingCopy{s, d, (size_t)len};
        }
        if (flags & EPB_FLAG_PIGGYBACK_ATOMIC) {
          const int k = ch_id < half ? 0 : 1;
          ds.sig[k] += 1;
          ds.sig_dirty[k] = true;
        }
        break;
      }
      case EPB_CMD_ATOMIC: {
        if (dof % 8 != 0 || dof + 8 > epb::kMetaBytes) {
          error(EPB_ERR_FAULT, (int64_t)((uint64_t)dst << 56 | dof));
          return;
        }
        flush(dst);  // the atomic follows the channel's earlier WRITEs to dst
        const uint64_t key = ((uint64_t)dst << 40) | dof;
        auto it = shadow.find(key);
        if (it == shadow.end()) it = shadow.emplace(key, seed_counter(dst, dof)).first;
        it->second += len;
        write_value(dst, dof, it->second);
        break;
      }
      case EPB_CMD_DRAIN: {
        flush_all();
        const int64_t upto = (int64_t)len - 1;
        if (len == 0 || cut == nullptr || upto >= idx) {
          wait_events(mark_streams(true));
        } else if (upto < cut_at) {
          // Idx was served in an earlier sweep: its copies completed before
          // that sweep's completion point; wait for everything issued up to now
          // only if that point is still in flight
          for (const Inflight& f : inflight) wait_events(f.evs);
        } else {
          wait_events(*cut);  // copies of commands <= Idx (cut taken right after Idx was served)
        }
        // mark the Drain completed (high-water mark)
        store_max_release(&ctx->fifo_host[cs.ch][EPB_CTL_COMPLETED], idx + 1);
        break;
      }
      case EPB_CMD_BARRIER: {
        flush_all();
        wait_events(mark_streams(true));
        const double timeout_s = (double)ctx->timeout_ns * 1e-9;
        if (!ctx->barrier) error(EPB_ERR_CONNECTION, 0xba);
        else if (epb_barrier_wait(ctx->barrier, (flags & EPB_FLAG_SAME_RAIL_BARRIER) != 0, timeout_s) != EPB_OK)
          error(EPB_ERR_DEADLOCK, 0xbb);
        store_max_release(&ctx->fifo_host[cs.ch][EPB_CTL_COMPLETED], idx + 1);
        break;
      }
      default:
        error(EPB_ERR_UNSUPPORTED, kind);
        break;
    }
  }

  void run() {
    if (!ok(cudaSetDevice(ctx->device))) return;
    const int C = ctx->cfg.fifo_channels;
    const int64_t cap = ctx->cfg.fifo_capacity, mask = cap - 1;
    dests.resize(ctx->world);
    for (int ch = 0; ch < C; ++ch) {
      if (epb::proxy_thread_of(ch, half, nthreads, ctx->proxy_chmap) != tid) continue;
      ChanState cs;
      cs.ch = ch;
      cs.head = load_acquire(&ctx->fifo_host[ch][EPB_CTL_HEAD]);
      cs.served_upto = cs.head;
      chans.push_back(cs);
    }
    // warm up each destination's copy path now (one 16-byte copy on its stream):
    // the first device-to-device copy of a process loads the driver's copy
    // kernel lazily, and that load waited for the LL kernel spinning on the
    // very copy (observed: the first proxy call of a fresh process timed out)
    // The same holds for the first value write to a peer mapping (its first
    // LL call stalled for seconds at EP=2 until both paths were warmed here).
    const size_t probe = epb::kMetaBytes + offsetof(epb::Scratch, trace) + sizeof(int64_t) * 62;
    // transfer engine: SM copy kernels by default (EP=4: LL pair 121 against 138 us,
    // HT proxy dispatch / combine 492 / 541 against 594 / 717 us with the copy
    // engine; profiles/r02_proxy_engine_n4.txt); EPB_PROXY_ENGINE=ce selects the
    // copy engine (cudaMemcpyAsync + cuStreamWriteValue64)
    sm_engine = true;
    if (const char* e = std::getenv("EPB_PROXY_ENGINE")) sm_engine = std::strcmp(e, "ce") != 0;
    if (const char* e = std::getenv("EPB_PCOPY_BLOCK_KB")) pcopy_block = std::max<int64_t>(1, std::atoll(e)) << 10;
    if (sm_engine) {  // the copy-kernel stream, its tickets, and one warm-up launch
      ok(cudaStreamCreateWithFlags(&kst, cudaStreamNonBlocking));
      if (ok(cudaMalloc(&tickets, sizeof(uint32_t) * kPcopyJobs))) ok(cudaMemset(tickets, 0, sizeof(uint32_t) * kPcopyJobs));
      if (tracing && ok(cudaMalloc(&stamps, sizeof(int64_t) * 4 * kStampRing)))
        ok(cudaMemset(stamps, 0, sizeof(int64_t) * 4 * kStampRing));
      PJob w;
      w.dest = ctx->rank;
      w.segs.push_back({ctx->base + probe, ctx->base + probe, 16});  // 16 bytes onto themselves
      w.bytes = 16;
      jobs.push_back(w);
      launch_jobs();
      ok(cudaStreamSynchronize(kst));
      kst_used = false;
    }
    for (int d = 0; d < ctx->world; ++d) {
      if (!ctx->peer[d]) continue;
      DestState& ds = dest(d);
      const size_t big = std::min<size_t>(ctx->cfg.ll_bytes, (size_t)1 << 20);
      const size_t src = ctx->ll_off(), dst = ctx->ll_off() + (d == ctx->rank ? big : 0);
      bool good = ok(cudaMemcpyAsync(ctx->peer[d] + probe, ctx->base + probe, 16, cudaMemcpyDefault, ds.st));
      if (good && big > 0 && d != ctx->rank)  // an LL-sized copy into the peer's (idle) LL region
        good = ok(cudaMemcpyAsync(ctx->peer[d] + dst, ctx->base + src, big, cudaMemcpyDefault, ds.st));
      if (good && write_value64())
        write_value64()(reinterpret_cast<CUstream>(ds.st), reinterpret_cast<CUdeviceptr>(ctx->peer[d] + probe), 0, 0);
      if (good) ok(cudaStreamSynchronize(ds.st));
    }
    // piggyback counters continue from their device values (proxy restarts)
    for (int d = 0; d < ctx->world; ++d)
      for (int k = 0; k < 2; ++k) {
        const size_t idx = (size_t)(k * 32 + tid) * epb::kMaxRanks + ctx->rank;
        if (ctx->peer[d]) dests[d].sig[k] = seed_counter(d, offsetof(epb::Meta, proxy_sig) + sizeof(uint64_t) * idx);
      }
    px->ready.fetch_add(1);
    int64_t idle = 0;
    std::vector<std::pair<int, int64_t>> served;
    while (!px->stop.load(std::memory_order_relaxed)) {
      bool any = false;
      served.clear();
      for (ChanState& cs : chans) {
        int64_t* ctl = ctx->fifo_host[cs.ch];
        const int64_t tail = load_acquire(&ctl[EPB_CTL_TAIL]);
        if (tail == cs.head) continue;
        tr(1, cs.ch, tail);
        // a DRAIN(Idx) in this batch: cut the copies right after command Idx
        int64_t cut_at = -1;
        for (int64_t i = cs.head; i < tail; ++i) {
          const int64_t s = EPB_CTL_SLOT0 + 2 * (i & mask);
          const uint64_t lo = (uint64_t)ctl[s], hi = (uint64_t)ctl[s + 1];
          const uint64_t l = (hi >> 20) & 0xFFFFFFFFull;
          if ((lo & 3) == EPB_CMD_DRAIN && l > 0 && (int64_t)l - 1 >= cs.head && (int64_t)l - 1 < i)
            cut_at = std::max(cut_at, (int64_t)l - 1);
        }
        std::vector<cudaEvent_t> cut;
        while (cs.head < tail) {
          const int64_t s = EPB_CTL_SLOT0 + 2 * (cs.head & mask);
          const uint64_t lo = (uint64_t)ctl[s], hi = (uint64_t)ctl[s + 1];
          const int64_t idx = cs.head++;
          serve(cs, idx, lo, hi, &cut, cs.served_upto);
          if (idx == cut_at) {
            flush_all();
            cut = mark_streams(true);
          }
        }
        cs.served_upto = cs.head;
        store_release(&ctl[EPB_CTL_HEAD], cs.head);
        for (cudaEvent_t ev : cut) pool.push_back(ev);  // (completed: waited on by the Drain)
        served.emplace_back(cs.ch, cs.head);
        any = true;
      }
      if (!served.empty()) {
        flush_all();
        if (px->count_only.load(std::memory_order_relaxed)) {
          for (auto& m : served) store_max_release(&ctx->fifo_host[m.first][EPB_CTL_COMPLETED], m.second);
        } else {
          Inflight f;
          f.evs = mark_streams(false);
          f.marks = served;
          inflight.push_back(std::move(f));
        }
      }
      while (!inflight.empty()) {
        Inflight& f = inflight.front();
        bool done = true;
        for (cudaEvent_t ev : f.evs) {
          const cudaError_t q = cudaEventQuery(ev);
          if (q == cudaErrorNotReady) {
            done = false;
            break;
          }
          if (!ok(q)) break;
        }
        if (!done) break;
        for (auto& m : f.marks) {
          store_max_release(&ctx->fifo_host[m.first][EPB_CTL_COMPLETED], m.second);
          tr(4, m.first, m.second);
        }
        for (cudaEvent_t ev : f.evs) pool.push_back(ev);
        inflight.pop_front();
      }
      if (!inflight.empty()) any = true;
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
    for (DestState& ds : dests)
      if (ds.st) cudaStreamSynchronize(ds.st);
    for (Inflight& f : inflight)
      for (cudaEvent_t ev : f.evs) cudaEventDestroy(ev);
    for (cudaEvent_t ev : pool) cudaEventDestroy(ev);
    for (DestState& ds : dests)
      if (ds.st) cudaStreamDestroy(ds.st);
    if (kst) {
      cudaStreamSynchronize(kst);
      cudaStreamDestroy(kst);
    }
    if (stamps) {  // device stamps (GPU clock) as trace kinds 10 (copy kernel start) / 11 (last signal)
      // kinds 10: kernel start, 11: last signal, 12: last block start, 13: last block's copies done
      std::vector<int64_t> h(4 * kStampRing);
      if (cudaMemcpy(h.data(), stamps, sizeof(int64_t) * h.size(), cudaMemcpyDeviceToHost) == cudaSuccess)
        for (int i = 0; i < kStampRing; ++i)
          for (int q = 0; q < 4; ++q)
            if (h[4 * i + q]) trace.push_back({h[4 * i + q], 10 + q, tid, i});
      cudaFree(stamps);
    }
    if (tickets) cudaFree(tickets);
    std::lock_guard<std::mutex> g(px->trace_m);
    px->trace.insert(px->trace.end(), trace.begin(), trace.end());
  }
};

void proxy_main(epb_proxy* px, int tid, int nthreads) {
  Worker w;
  w.px = px;
  w.ctx = px->ctx;
  w.tid = tid;
  w.nthreads = nthreads;
  w.half = std::max(1, px->ctx->cfg.fifo_channels / 2);
  w.tracing = px->ctx->trace != 0;
  w.run();
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

int epb_proxy_nthreads(const epb_ctx* ctx) {
  return std::max(1, std::min({ctx->cfg.proxy_threads, ctx->cfg.fifo_channels, 32}));
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
  if (!write_value64()) return epb_set_error(EPB_ERR_CUDA, "cuStreamWriteValue64 is not available from the driver");
  const int n = epb_proxy_nthreads(ctx);
  epb_proxy* px = new epb_proxy();
  px->ctx = ctx;
  for (int i = 0; i < n; ++i) px->threads.emplace_back(proxy_main, px, i, n);
  ctx->proxy = px;
  // no kernel may depend on the proxy before its copy paths are warm
  const auto t0 = std::chrono::steady_clock::now();
  while (px->ready.load() < n && std::chrono::steady_clock::now() - t0 < std::chrono::seconds(60))
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  return EPB_OK;
}

extern "C" int epb_proxy_stop(epb_t* ctx) {
  if (!ctx || !ctx->proxy) return EPB_OK;
  ctx->proxy->stop.store(true);
  for (auto& t : ctx->proxy->threads) t.join();
  {  // keep the threads' trace events for epb_proxy_trace
    auto& tv = ctx->proxy->trace;
    std::sort(tv.begin(), tv.end(), [](const TraceEv& x, const TraceEv& y) { return x.t_ns < y.t_ns; });
    ctx->proxy_trace.clear();
    for (const TraceEv& e : tv) ctx->proxy_trace.insert(ctx->proxy_trace.end(), {e.t_ns, e.kind, e.a, e.b});
  }
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

// Trace events of the last STOPPED proxy (the threads hand theirs over at
// exit): rows of {host CLOCK_REALTIME ns, kind, a, b}; kind 1 = new tail seen
// (a = channel, b = tail), 2 = copy issued (a = dst, b = bytes), 3 = value write
// issued (a = dst, b = value), 4 = COMPLETED published (a = channel, b = value);
// API-cost markers: 6 = before the copy call, 7 = before the value write,
// 8 / 9 = around a completion-event record.  Returns the number of events.
extern "C" int64_t epb_proxy_trace(epb_t* ctx, int64_t* out, int64_t max_events) {
  if (!ctx) return 0;
  const int64_t n = (int64_t)ctx->proxy_trace.size() / 4;
  if (out) std::memcpy(out, ctx->proxy_trace.data(), sizeof(int64_t) * 4 * std::min(n, std::max<int64_t>(0, max_events)));
  return n;
}
