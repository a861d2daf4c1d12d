// common.cuh — shared device/host definitions for the sm_100a EP kernels.
//
// Memory model used throughout ("release/acquire discipline"):
//   * payload rows go to peer memory with plain 16-byte stores (NVLink posted
//     writes); a block barrier orders all of a block's stores before ONE
//     red.release.sys on the destination's counter (release cumulativity);
//   * receivers spin with ld.acquire.sys on their own counter words, then a
//     block barrier publishes the observation to the rest of the block;
//   * small control messages (dispatch counts, combine mode, host counts) are
//     TAGGED words: value << 32 | call epoch, one naturally aligned 8-byte
//     store each (single-copy atomic), so the data is its own flag — no
//     fence on the writer, no flag round trip for the reader.
// This replaces the reference ring's plain loads/stores (kernels.py:5-8,
// kernels.py:67-79), which rely on x86-TSO and do not carry over to a
// GPU <-> peer / GPU <-> host channel.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/epb.h"

namespace epb {

constexpr int kMaxRanks = EPB_MAX_RANKS;
constexpr int kMaxLocal = EPB_MAX_LOCAL;
constexpr int kMaxChannels = EPB_MAX_CHANNELS;
constexpr int kMaxLocalExperts = EPB_MAX_LOCAL_EXPERTS;
constexpr int kMaxFifo = 64;  // 6-bit channel_id (command.py:37)
constexpr int kMaxLanes = 80;  // chunked-ring transport: lanes (sender/receiver block pairs)

// ---------------------------------------------------------------------------
// Symmetric-region layout (identical offsets on every rank).
//   [0, kMetaBytes)                 Meta: flags/counters/mailboxes peers write
//   [kMetaBytes, kRegionHeader)     Scratch: this rank's private plan words
//   [kRegionHeader, +nvl_bytes)     normal-mode arena (recv slots + staging)
//   [.., +ll_bytes)                 low-latency region
// ---------------------------------------------------------------------------
// Tagged word helpers: value << 32 | epoch (see the memory-model note).
constexpr uint32_t kNotifyAbort = 0xffffffffu;  // "no value" (aborted call, not in region, ...)
__host__ __device__ constexpr uint64_t tagged(uint32_t value, uint32_t epoch) {
  return ((uint64_t)value << 32) | epoch;
}

struct NotifyMsg {                          // one source rank's dispatch counts (tagged words)
  uint64_t counts_per_rank[kMaxRanks];      // src's num_tokens_per_rank
  uint64_t slot;                            // src's receive slot (where peers write TO src)
  uint64_t pad[7];
  uint64_t channel_counts[kMaxChannels];    // src's tokens to me, per channel
  uint64_t expert_counts[kMaxLocalExperts]; // src's tokens for each of my local experts
};

struct Meta {
  uint32_t disp_done[kMaxRanks];         // += 1 per dispatch block of src (monotonic)
  uint32_t comb_done[kMaxRanks];         // += 1 per combine block of src (monotonic)
  // LL direct transport: += 1 per sender block of src once its rows (and, for
  // block 0, the count header) have landed.  Cumulative per parity: the
  // receiver waits for (calls of this parity so far) x (grid width), so every
  // rank must keep the same LL grid width for the life of the context
  // (ll_blocks pins it at the first call)
  uint32_t ll_disp_cnt[2][kMaxRanks];
  uint32_t ll_comb_cnt[2][kMaxRanks];
  // CPU-proxy signals (proxy.cpp): proxy_sig[kind * 32 + t][src] = how many
  // piggybacked WRITEs src's proxy thread t has landed here, cumulative; kind
  // 0 = LL dispatch channels, 1 = LL combine channels.  Written with
  // stream-ordered value stores after the copies they count.
  uint64_t proxy_sig[kMaxFifo][kMaxRanks];
  uint64_t ht_sig[2][kMaxRanks];         // proxy HT transport: src's ATOMIC += 1 per [dispatch|combine] call
  // combine mode message (tagged words): where src's input rows / weights live
  // inside src's region, in 16-byte / 4-byte units (kNotifyAbort: not there)
  uint64_t comb_msg[2][kMaxRanks][2];
  // chunked rings (chunked.cu), cumulative token counts, [dispatch|combine]:
  // rc_tail[.][src][lane]: slots src has filled in its ring here (producer-advanced)
  // rc_head[.][dst][lane]: slots dst has drained from my ring there (credit return)
  uint32_t rc_tail[2][kMaxRanks][kMaxLanes];
  uint32_t rc_head[2][kMaxRanks][kMaxLanes];
  NotifyMsg mbox[2][kMaxRanks];
};

struct Scratch {                         // private to the owning rank
  int32_t abort;                         // the last dispatch aborted (combine skips its data path)
  uint32_t pad0[3];
  // dispatch, between the blocks of one rank (tagged words, this call's epoch):
  uint64_t ch_cnt[kMaxRanks][kMaxChannels];   // my tokens per (destination, channel)
  uint64_t ch_excl[kMaxRanks][kMaxChannels];  // exclusive prefix over channels of ch_cnt
  // plan[0][d]: d's receive slot (kNotifyAbort: aborted), [1][d]: my first row
  // at d, [2][d]: rows I send to d, [3][d]: where they start in my send
  // staging (proxy transport)
  uint64_t plan[4][kMaxRanks];
  uint32_t ll_ticket[4];                 // LL last-warp tickets: [dispatch|combine][parity]
  // chunked rings: this rank's own cumulative positions, [dispatch|combine]
  uint32_t rc_sent[2][kMaxRanks][kMaxLanes];   // slots I have filled in dst's ring
  uint32_t rc_recvd[2][kMaxRanks][kMaxLanes];  // slots I have drained from src's ring
  // LL epochs live on the device (bumped by each call's last warp) so LL calls
  // can be captured in CUDA graphs and replayed: [dispatch|combine]
  uint32_t ll_epoch[2];
  uint32_t ll_pcnt[2];                   // proxy-transport calls so far (signal targets)
  // LL proxy transport: arrivals per command group [dispatch|combine][parity][group];
  // the add that completes a group pushes its WRITE; the call's last block
  // (ticket) zeroes its parity's counters, so a call that aborted half-way
  // cannot leave stale arrivals for the calls after it
  uint32_t llp_grp[2][2][kMaxFifo];
  // LL proxy transport, rows to myself: stored straight into my receive block
  // (no loopback through the proxy); += 1 per completed group [dispatch|combine]
  uint32_t llp_self[2];
  // LL proxy transport, leader polling (EPB_LL_POLL_LEADER): block 0 waits for
  // the proxies' signals and publishes the call count here for the other blocks
  uint32_t llp_go[2];
  // normal-mode call epochs and cumulative done targets [dispatch|combine],
  // device-resident so a layout -> dispatch -> combine step can be captured in
  // a CUDA graph and replayed: each call reads them at kernel start and its
  // last block (norm_ticket) stores the new values (norm_call_begin / _end)
  uint32_t norm_epoch[2];
  uint32_t norm_cum[2];
  uint32_t norm_ticket[2];
  // GPU -> CPU FIFOs: control arrays live in pinned host memory; the producer
  // keeps its tail (and a cached head) here, in device memory.
  uint64_t fifo_ctl[kMaxFifo];           // device aliases of the pinned ctl arrays
  int64_t fifo_tail[kMaxFifo];
  int64_t fifo_head[kMaxFifo];
  int32_t fifo_channels;
  int32_t fifo_cap;
  // phase timestamps (%globaltimer ns) written by block 0 / thread 0 when
  // tracing is enabled (EPB_TRACE=1); read with epb_trace()
  int64_t trace[64];
};

constexpr size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
constexpr size_t kMetaBytes = align_up(sizeof(Meta), 4096);
constexpr size_t kScratchBytes = align_up(sizeof(Scratch), 4096);
constexpr size_t kRegionHeader = kMetaBytes + kScratchBytes;

#ifdef __CUDACC__
#define EPB_HD __host__ __device__
#else
#define EPB_HD
#endif
// FIFO channel -> CPU proxy thread, shared by the proxy (which channels a thread
// serves) and the LL receivers (whose signal words to wait on).  0: c % nth.
// 1 ("phase", EPB_PROXY_CHMAP=phase): every channel of the first half (LL
// dispatch) on thread 0, of the second half (LL combine) on thread 1 % nth, so
// one thread sees all of a phase's commands in one sweep and issues them together.
EPB_HD inline int proxy_thread_of(int ch, int half, int nth, int mode) {
  if (mode == 1) return ch < half ? 0 : 1 % nth;
  return ch % nth;
}


// Pinned, device-mapped host words the kernels publish to the CPU.
// The dispatch publishes the receive counts to the host as tagged words, so
// the host needs no flag and the kernel no system-scope fence (a fence.sys
// would queue behind the copy warps' NVLink traffic on the SM).
// notify[0] = number of received rows (kNotifyAbort if the call aborted),
// notify[1 + e] = rows for local expert e (padded to expert_alignment).
struct HostInfo {
  volatile int64_t err_code;
  volatile int64_t err_detail;
  volatile uint64_t notify[1 + kMaxLocalExperts];
};

// What a kernel needs to know about one (possibly emulated) rank.
struct RankView {
  int rank, world;
  char* base;                  // my region
  char* peer[kMaxRanks];       // every rank's region, mapped in this process
  HostInfo* host;              // device alias of the pinned HostInfo
  uint64_t timeout_ns;
  int trace;                   // record phase timestamps into Scratch::trace
  uint64_t region_bytes;       // size of every rank's region
};

__host__ __device__ inline Meta* meta_of(char* base) { return reinterpret_cast<Meta*>(base); }
__host__ __device__ inline Scratch* scratch_of(char* base) { return reinterpret_cast<Scratch*>(base + kMetaBytes); }

// ---------------------------------------------------------------------------
// PTX helpers (sm_100a).
// ---------------------------------------------------------------------------
#ifdef __CUDACC__
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(volatile uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const volatile uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int64_t ld_volatile(const int64_t* p) {
  int64_t v;
  asm volatile("ld.volatile.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Release/acquire fence at system scope.  fence.sc is not needed anywhere on
// this path (no store->load ordering across different flags is relied on) and
// is far more expensive when many threads execute it.
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// 16-byte streaming loads/stores.  Source rows are read once: keep them out
// of L1.  Peer stores are plain st.global (they leave the SM as NVLink writes).
__device__ __forceinline__ int4 ld_nc_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_cg_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_na_v4(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA engine) helpers: cp.async.bulk global -> shared with an
// mbarrier transaction count, shared -> global in bulk groups (SASS UBLKCP).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_u32(smem)),
               "r"(bytes)
               : "memory");
}
// bulk store with an L2 eviction-priority hint (keep the rows L2-resident for
// the kernel that reads them next, like the plain stores' write-allocate)
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_store_hint(void* gmem, const void* smem, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gmem),
               "r"(smem_u32(smem)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");  // async-proxy writes before generic releases
}
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Phase timestamp for tracing (first thread of the first block of the rank).
__device__ __forceinline__ void trace_mark(const RankView& rv, int idx) {
  if (rv.trace && threadIdx.x == 0 && blockIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    scratch_of(rv.base)->trace[idx] = (int64_t)t;
  }
}
// Latest time any block reached this point (thread 0 of every block).
__device__ __forceinline__ void trace_mark_max(const RankView& rv, int idx) {
  if (rv.trace && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(reinterpret_cast<unsigned long long*>(&scratch_of(rv.base)->trace[idx]), (unsigned long long)t);
  }
}

// Latest time any thread passed this point (the calling thread only).
__device__ __forceinline__ void trace_mark_max_any(const RankView& rv, int idx) {
  if (rv.trace) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(reinterpret_cast<unsigned long long*>(&scratch_of(rv.base)->trace[idx]), (unsigned long long)t);
  }
}

// gpu-scope acq_rel fetch-add (the last-arriver ticket pattern: each arriving
// warp releases its prior stores, the winner acquires all of them and its own
// sys-scope release then covers them by cumulativity).
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// In-place scan of n ints in shared memory by one warp (exclusive or
// inclusive); returns the total.  Each lane owns a contiguous run of
// ceil(n/32) elements, so the dependent chain is n/32 + 5 steps.
__device__ __forceinline__ int warp_scan_smem(int32_t* a, int n, int lane, bool exclusive) {
  const int per = (n + 31) / 32, base = lane * per;
  int local = 0;
  for (int i = 0; i < per; ++i)
    if (base + i < n) local += a[base + i];
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  int run = incl - local;
  for (int i = 0; i < per; ++i) {
    if (base + i < n) {
      const int v = a[base + i];
      a[base + i] = exclusive ? run : run + v;
      run += v;
    }
  }
  return __shfl_sync(0xffffffffu, incl, 31);
}

// Normal-mode call bookkeeping (Scratch::norm_*).  begin: thread 0 reads the
// previous call's epoch and cumulative target; every block derives this
// call's values (epoch + 1, cum + grid width).  end: the last block of the
// grid (gpu-scope ticket: every block has read the old values by then)
// stores them for the next call on the stream.
__device__ __forceinline__ void norm_call_begin(const RankView& rv, int kind, uint32_t grid, uint32_t* epoch,
                                                uint32_t* target) {
  Scratch* sc = scratch_of(rv.base);
  *epoch = *reinterpret_cast<volatile uint32_t*>(&sc->norm_epoch[kind]) + 1u;
  *target = *reinterpret_cast<volatile uint32_t*>(&sc->norm_cum[kind]) + grid;
}
__device__ __forceinline__ void norm_call_end(const RankView& rv, int kind, uint32_t epoch, uint32_t target) {
  Scratch* sc = scratch_of(rv.base);
  if (atom_add_acq_rel_gpu(&sc->norm_ticket[kind], 1u) == gridDim.x - 1) {
    sc->norm_ticket[kind] = 0;
    *reinterpret_cast<volatile uint32_t*>(&sc->norm_epoch[kind]) = epoch;
    *reinterpret_cast<volatile uint32_t*>(&sc->norm_cum[kind]) = target;
  }
}

// Record an error into the host-visible word (first error wins is not
// required: any non-zero code makes the host raise).
__device__ __forceinline__ void report_error(const RankView& rv, int code, int64_t detail) {
  rv.host->err_detail = detail;
  rv.host->err_code = code;
  scratch_of(rv.base)->abort = code;
  __threadfence_system();
}

// Spin until *p >= target (wrap-safe for monotonically increasing u32
// counters).  Returns false on timeout after reporting EPB_ERR_DEADLOCK.
// max_sleep_ns > 0: back off with __nanosleep (doubling from 32 ns) between
// polls, for waits many warps run at once so polling does not steal L2 and
// issue bandwidth from the warps doing the work.
__device__ __forceinline__ bool wait_geq(const RankView& rv, const uint32_t* p, uint32_t target, int64_t tag,
                                         unsigned max_sleep_ns = 0) {
  uint64_t t0 = 0;
  int iter = 0;
  unsigned sleep_ns = 32;
  while (static_cast<int32_t>(ld_acquire_sys(p) - target) < 0) {
    if (max_sleep_ns) {
      __nanosleep(sleep_ns);
      sleep_ns = min(sleep_ns * 2, max_sleep_ns);
    }
    if ((++iter & 1023) == 0) {
      uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > rv.timeout_ns) {
        report_error(rv, EPB_ERR_DEADLOCK, tag);
        return false;
      }
    }
  }
  return true;
}
// Spin until the tagged word *p carries `epoch`; returns its value, or
// kNotifyAbort after reporting EPB_ERR_DEADLOCK on timeout.
// sleep_ns > 0: __nanosleep between polls (for waits many blocks run at once).
__device__ __forceinline__ uint32_t wait_tagged(const RankView& rv, const uint64_t* p, uint32_t epoch, int64_t tag,
                                                unsigned sleep_ns = 0) {
  uint64_t t0 = 0;
  int iter = 0;
  while (true) {
    const uint64_t v = ld_relaxed_sys(p);
    if ((uint32_t)v == epoch) return (uint32_t)(v >> 32);
    if (sleep_ns) __nanosleep(sleep_ns);
    if ((++iter & 1023) == 0) {
      const uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > rv.timeout_ns) {
        report_error(rv, EPB_ERR_DEADLOCK, tag);
        return kNotifyAbort;
      }
    }
  }
}
// Same as wait_geq, for a counter written only by this GPU (gpu-scope acquire).
__device__ __forceinline__ bool wait_geq_gpu(const RankView& rv, const uint32_t* p, uint32_t target, int64_t tag,
                                             unsigned sleep_ns = 0) {
  uint64_t t0 = 0;
  int iter = 0;
  while (static_cast<int32_t>(ld_acquire_gpu(p) - target) < 0) {
    if (sleep_ns) __nanosleep(sleep_ns);
    if ((++iter & 1023) == 0) {
      uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > rv.timeout_ns) {
        report_error(rv, EPB_ERR_DEADLOCK, tag);
        return false;
      }
    }
  }
  return true;
}
// sleep_ns > 0: __nanosleep between polls (counters written by a copy engine
// on the proxy's behalf: a tight acquire loop on the line it writes slows it).
__device__ __forceinline__ bool wait_geq64(const RankView& rv, const uint64_t* p, uint64_t target, int64_t tag,
                                           unsigned sleep_ns = 0) {
  uint64_t t0 = 0;
  int iter = 0;
  while (static_cast<int64_t>(ld_acquire_sys(p) - target) < 0) {
    if (sleep_ns) __nanosleep(sleep_ns);
    if ((++iter & 1023) == 0) {
      uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > rv.timeout_ns) {
        report_error(rv, EPB_ERR_DEADLOCK, tag);
        return false;
      }
    }
  }
  return true;
}
#endif  // __CUDACC__

}  // namespace epb
