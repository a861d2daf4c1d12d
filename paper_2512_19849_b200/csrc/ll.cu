// ll.cu — low-latency (decode) EP path on sm_100a.
//
//   ll_dispatch : one message per (token, expert), no dedup (SPEC.md:426-434,
//                 :463), fused FP8 e4m3 quantisation per 128 channels,
//                 deterministic slots (rank of the token among the source's
//                 tokens for that expert), completion counted per sender
//                 block (the LL fence of PAPER.md:343-346 / kernels.py:187-248
//                 collapses to "all X writes, then the count": each block's
//                 red.release.sys covers its rows, block 0's also the count
//                 header, and the receiver acquires the per-source counter).
//   ll_combine  : expert outputs pushed back to the source, weighted top-k
//                 reduce in fp32 in ascending top-k order.
//
// Two transports share the same receive layout (ll_common.cuh):
//   direct : the kernel stores rows into the peer's receive block over NVLink;
//   proxy  : the kernel stores rows into its local send block (same layout)
//            and one producer lane pushes 16-byte TransferCmds (command.py
//            layout) into a pinned-host FIFO (kernels.py:23-31 ctl layout);
//            CPU proxy threads (proxy.cpp) coalesce the WRITEs into copies and
//            execute the piggybacked atomic as a stream-ordered counter bump.
//
// Latency structure: every phase is split into many small warp work items
// ((token, 512-channel chunk) for the quantise+scatter, one row per warp with
// 8 x 16 B loads in flight per lane for the copies) so a 128-token batch
// spreads over all SMs.  Epochs live on the device so a dispatch/combine pair
// can be captured in a CUDA graph and replayed.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ctx.h"
#include "ll_common.cuh"

namespace epb {

constexpr int kChunkCh = 512;  // channels per (token, chunk) item: 32 lanes x 16 channels

// standalone per-token cast (warp per (token, chunk))
__global__ void __launch_bounds__(kLLThreads) fp8_cast_kernel(const __nv_bfloat16* __restrict__ x, int T, int H,
                                                               int round_scale, uint8_t* __restrict__ q,
                                                               float* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int S = H / 128, NCH = (H + kChunkCh - 1) / kChunkCh;
  for (int item = gw; item < T * NCH; item += nw) {
    const int t = item / NCH, ch0 = (item % NCH) * kChunkCh + lane * 16;
    const int4* src = reinterpret_cast<const int4*>(x + (size_t)t * H);
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

// Warp copy of n16 16-byte words with 8 loads in flight per lane.  kNc selects
// the non-coherent path (read-only inputs); data written by peers during the
// kernel is read with ld.global.cg.
template <bool kNc>
__device__ __forceinline__ void warp_copy(const int4* src, int4* dst, int n16, int lane) {
  constexpr int U = 8;
  for (int base = lane; base < n16; base += 32 * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * u;
      if (i < n16) v[u] = kNc ? ld_nc_v4(src + i) : ld_cg_v4(src + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * u;
      if (i < n16) st_v4(dst + i, v[u]);
    }
  }
}

__device__ __forceinline__ int ordinal_of(const uint32_t* bm_row, int t) {
  const int w = t >> 5;
  int c = 0;
  for (int i = 0; i < w; ++i) c += __popc(bm_row[i]);
  return c + __popc(bm_row[w] & ((1u << (t & 31)) - 1u));
}

// ---------------------------------------------------------------------------
// Proxy transport: command groups.  Group g (< G = disp_channels, one FIFO
// channel each) owns chunk c = g / R of destination d = g % R's rows (rows
// [c*n/nc, (c+1)*n/nc) of the n rows for d, nc = chunks of d).  The warp whose
// arrival completes a group pushes that group's WRITE at once — while other
// groups are still being produced (token-level GPU-initiated commands,
// PAPER.md:136-140, :339); nothing waits for the whole grid.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int group_chunks(int G, int R, int d) { return (G - d + R - 1) / R; }

__device__ __forceinline__ int group_of_row(const int32_t* s_g1, int G, int R, int d, int row) {
  const int nc = group_chunks(G, R, d);
  for (int c = 0; c < nc; ++c)
    if (row < s_g1[d + R * c]) return d + R * c;
  return d + R * (nc - 1);
}

// Receiver side: piggybacked WRITEs from src's proxy thread pt to me per call
// (group b goes to rank b % R on channel chan0 + b, served by proxy_thread_of).
__device__ __forceinline__ int proxy_cmds_per_call(int G, int R, int me, int chan0, int half, int nth, int mode,
                                                   int pt) {
  int n = 0;
  for (int b = me; b < G; b += R) n += proxy_thread_of(chan0 + b, half, nth, mode) == pt;
  return n;
}

// one thread: wait until every source's proxy threads have landed this call's groups
// (my own rows never go through the proxy: they were stored locally and
// counted on Scratch::llp_self — one add per group, G / R groups per call)
__device__ __forceinline__ void wait_proxy_groups(const RankView& rv, const Meta* my, int kind, int G, int half, int R,
                                                  int me, int nth, int chmap, uint64_t calls, int64_t tag,
                                                  unsigned poll_ns) {
  for (int i = threadIdx.x; i < R * nth; i += blockDim.x) {
    const int s = i / nth, pt = i % nth;
    if (s == me) {
      if (pt == 0)
        wait_geq_gpu(rv, &scratch_of(rv.base)->llp_self[kind], (uint32_t)(calls * (uint64_t)(G / R)), tag + i);
      continue;
    }
    const int n = proxy_cmds_per_call(G, R, me, kind ? half : 0, half, nth, chmap, pt);
    if (n > 0) wait_geq64(rv, &my->proxy_sig[kind * 32 + pt][s], calls * (uint64_t)n, tag + i, poll_ns);
  }
}

// The receive wait of the proxy transport.  Default: every block polls the
// signal words.  leader: block 0 alone polls them (fewer pollers on the lines
// the copy engines write) and releases the call count to the other blocks.
// The caller synchronises the block afterwards.
__device__ __forceinline__ void wait_proxy_recv(const RankView& rv, const Meta* my, int kind, int G, int half, int R,
                                                int me, int nth, int chmap, uint64_t calls, int64_t tag, int poll_ns,
                                                int leader) {
  if (!leader) {
    wait_proxy_groups(rv, my, kind, G, half, R, me, nth, chmap, calls, tag, (unsigned)poll_ns);
    return;
  }
  Scratch* sc = scratch_of(rv.base);
  if (blockIdx.x == 0) {
    wait_proxy_groups(rv, my, kind, G, half, R, me, nth, chmap, calls, tag, (unsigned)poll_ns);
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(&sc->llp_go[kind], (uint32_t)calls);
  } else if (threadIdx.x == 0) {
    wait_geq_gpu(rv, &sc->llp_go[kind], (uint32_t)calls, tag + 0x3f, (unsigned)poll_ns);
  }
}

// ---------------------------------------------------------------------------
// LL dispatch
// ---------------------------------------------------------------------------
struct LLDispatchParams {
  int n_local, phases, use_proxy, disp_channels, pthreads;
  int ngroups;  // proxy transport: command groups (R x groups per destination, <= disp_channels)
  int poll_ns, poll_leader;  // proxy transport receive polling (ll_poll)
  int chmap;                 // proxy_thread_of mode of the channels' proxy threads
  RankView rv[kMaxLocal];
  epb_ll_dispatch_args_t a[kMaxLocal];
  LLGeom g;
  int64_t ll_off;
};

// Send-block reuse.  A call writes the send blocks of its parity, which the
// proxy's copies of the call two back read.  Those copies are complete by
// causality: this rank's previous call (other parity) could only finish its
// receive after every peer's previous call pushed, and a peer pushes only
// after its own receive of the call two back — which waited for this rank's
// copies to land.  So no wait is needed as long as a call's receive runs
// before the send of the call two after it (DeepEP's double-buffer rule; the
// recv hook must be called in time).  Block 0 checks it with ONE read of the
// channel's COMPLETED word (pinned host memory — a read per block would queue
// ~150 PCIe reads: measured 125 us) and reports a violation.
__device__ __forceinline__ void check_channel_backlog(const RankView& rv, int ch, int64_t keep) {
  Scratch* sc = scratch_of(rv.base);
  const int64_t* ctl = reinterpret_cast<const int64_t*>(sc->fifo_ctl[ch]);
  const int64_t want = sc->fifo_tail[ch] - keep;  // all but the newest `keep` commands
  if (want > 0 && ld_acquire_sys(ctl + EPB_CTL_COMPLETED) < want)
    report_error(rv, EPB_ERR_PROTOCOL, ((int64_t)0x540 << 32) | ch);
}

// The single lane whose arrival completed dispatch group gid: one WRITE (the
// chunk-0 group from the block start: d's per-expert count header, written by
// block 0, whose arrival the group also awaits) with a piggybacked signal on
// FIFO channel gid (command.py layout, arena offsets).
__device__ __noinline__ void ll_push_dispatch_group(const LLDispatchParams& P, int lr, int gid, const int32_t* s_g0,
                                                    const int32_t* s_g1, uint32_t epoch) {
  const RankView& rv = P.rv[lr];
  const LLGeom& g = P.g;
  const int R = g.R, me = rv.rank, par = epoch & 1;
  const int d = gid % R, c = gid / R;
  Scratch* sc = scratch_of(rv.base);
  if (d == me) {  // my own rows (and header) are already in my receive block: count the group
    red_release_gpu_add(&sc->llp_self[0], 1u);
    return;
  }
  const int64_t send_blk = g.off_disp_send + (int64_t)(par * R + d) * g.disp_block;
  // no fence here: fifo_push's st.release.sys of TAIL is cumulative — it orders
  // the group's rows and header (acquired through the arrival counter) before
  // the command at system scope (a separate fence.sys cost 2.3 us)
  const int64_t rel = P.ll_off - (int64_t)kRegionHeader;  // commands address the arena start
  const int64_t first = c == 0 ? 0 : g.hdr_bytes + (int64_t)s_g0[gid] * g.disp_row;
  const int64_t len = (c == 0 ? g.hdr_bytes : 0) + (int64_t)(s_g1[gid] - s_g0[gid]) * g.disp_row;
  const int64_t dst_blk = g.off_disp_recv + (int64_t)(par * R + me) * g.disp_block;
  uint64_t lo, hi;
  cmd_pack_dev(EPB_CMD_WRITE, d, gid, rel + send_blk + first, rel + dst_blk + first, len, EPB_FLAG_PIGGYBACK_ATOMIC,
               lo, hi);
  fifo_push(rv, gid, lo, hi);
  if (rv.trace && gid < 12) scratch_of(rv.base)->trace[40 + gid] = (int64_t)globaltimer();
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
  char* my_ll = rv.base + P.ll_off;
  Scratch* sc = scratch_of(rv.base);
  Meta* my_meta = meta_of(rv.base);
  const uint32_t base_epoch = *reinterpret_cast<volatile uint32_t*>(&sc->ll_epoch[0]);
  const uint32_t base_pcnt = *reinterpret_cast<volatile uint32_t*>(&sc->ll_pcnt[0]);
  const bool sending = (P.phases & 1) != 0;
  const uint32_t epoch = sending ? base_epoch + 1 : base_epoch;
  const uint64_t pexp = base_pcnt + ((sending && P.use_proxy) ? 1 : 0);
  const int par = epoch & 1;
  const int64_t rstride = g.disp_row;
  const int meta_off = g.use_fp8 ? H + 4 * S : 2 * H;
  extern __shared__ uint8_t smem[];
  trace_mark(rv, 24);
  trace_mark_max(rv, 39);  // the last block to start

  if (sending) {
    const int W = max(1, (T + 31) / 32);
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem);
    int32_t* cnt = reinterpret_cast<int32_t*>(bm + (size_t)E * W);
    int32_t* pre = cnt + E;
    int16_t* s_e = reinterpret_cast<int16_t*>(pre + E);  // [T][k] expert ids (-1: masked), read by the items
    for (int i = tid; i < E * W; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    for (int i = tid; i < T * k; i += blockDim.x) {
      const int64_t e = a.topk_idx[i];
      const int t = i / k;
      const bool ok = e >= 0 && e < E;
      s_e[i] = ok ? (int16_t)e : (int16_t)-1;
      if (ok) atomicOr(&bm[(size_t)e * W + (t >> 5)], 1u << (t & 31));
    }
    __syncthreads();
    trace_mark(rv, 30);
    for (int e = tid; e < E; e += blockDim.x) {
      int c = 0;
      for (int w = 0; w < W; ++w) c += __popc(bm[(size_t)e * W + w]);
      cnt[e] = c;
      pre[e] = c;
    }
    __syncthreads();
    trace_mark(rv, 62);
    for (int d = warp; d < R; d += nw) warp_scan_smem(pre + d * L, L, lane, true);  // row of expert in dst block
    // proxy transport: token-major rows per destination (a contiguous token
    // range is a contiguous row range, so command groups are row ranges)
    int16_t* s_loc = s_e + (size_t)a.max_tokens * k;  // [T][k] slot of (t, j) among t's rows for d(e); < -1: dup
    int32_t* rs = reinterpret_cast<int32_t*>(s_loc + (size_t)a.max_tokens * k);  // [R][T+1] first row of t at d
    __shared__ int32_t s_g0[kMaxFifo], s_g1[kMaxFifo], s_gexp[kMaxFifo];
    __shared__ uint32_t s_arr[kMaxFifo];  // this block's arrivals per group
    const int G = P.ngroups;
    for (int gg = tid; gg < G; gg += blockDim.x) s_arr[gg] = 0;
    if (P.use_proxy) {
      // per (token, top-k entry): its slot among the token's rows for the entry's
      // destination (rows = distinct experts, in top-k order), or -2 - j of the
      // entry j it duplicates.  One lane per entry, kp lanes per token; the
      // token's other entries come by shuffles (__match_any_sync measured
      // ~600 cycles per call here)
      for (int i = tid; i < R * (T + 1); i += blockDim.x) rs[i] = 0;
      __syncthreads();
      trace_mark(rv, 63);
      const int kp = k <= 1 ? 1 : 1 << (32 - __clz(k - 1));  // entries rounded to a power of two
      const int sub = lane / kp, j = lane % kp, l0 = sub * kp;
      for (int t0 = warp * (32 / kp); t0 < T; t0 += nw * (32 / kp)) {
        const int t = t0 + sub;
        const bool entry = t < T && j < k;
        const int e = entry ? s_e[t * k + j] : -1;
        int fl = j;  // the token's first entry holding e
        for (int jj = 0; jj < kp; ++jj) {
          const int ej = __shfl_sync(0xffffffffu, e, l0 + jj);
          if (fl == j && jj < j && ej == e) fl = jj;
        }
        const bool first = e >= 0 && fl == j;
        const int dd = first ? e / L : -1;
        int before = 0, tot = 0;  // first entries of the token for dd: before mine, all
        for (int jj = 0; jj < kp; ++jj) {
          const int dj = __shfl_sync(0xffffffffu, dd, l0 + jj);
          if (first && dj == dd) {
            ++tot;
            before += jj < j;
          }
        }
        if (first && before == 0) rs[dd * (T + 1) + t] = tot;
        if (entry) s_loc[t * k + j] = (int16_t)(first ? before : e < 0 ? -1 : -2 - fl);
      }
      __syncthreads();
      trace_mark(rv, 31);
      for (int d = warp; d < R; d += nw) warp_scan_smem(rs + d * (T + 1), T + 1, lane, true);
      __syncthreads();
      const int NCHc = (H + kChunkCh - 1) / kChunkCh;
      for (int gi = tid; gi < G; gi += blockDim.x) {
        const int d = gi % R, c = gi / R, nc = group_chunks(G, R, d);
        const int n = rs[d * (T + 1) + T];
        s_g0[gi] = (int)((int64_t)c * n / nc);
        s_g1[gi] = (int)((int64_t)(c + 1) * n / nc);
        // arrivals the group expects: each of its rows, once per chunk item,
        // and for chunk 0 block 0's header
        s_gexp[gi] = (s_g1[gi] - s_g0[gi]) * NCHc + (c == 0 ? 1 : 0);
      }
      if (blockIdx.x == 0) {
        // block 0 writes every destination's per-expert count header (all
        // threads; my own into my receive block) and reports it with its rows
        for (int i = tid; i < R * L; i += blockDim.x) {
          const int d = i / L;
          const int64_t blk = d == me ? g.off_disp_recv + (int64_t)(par * R + me) * g.disp_block
                                      : g.off_disp_send + (int64_t)(par * R + d) * g.disp_block;
          reinterpret_cast<int32_t*>(my_ll + blk)[i % L] = cnt[i];
        }
        for (int gg = tid; gg < R && gg < G; gg += blockDim.x) s_arr[gg] = 1;
      }
      __syncthreads();
      // empty groups (no rows, not chunk 0) still send their WRITE: every group
      // signals once per call
      if (blockIdx.x == 0)
        for (int gi = tid; gi < G; gi += blockDim.x)
          if (s_gexp[gi] == 0) ll_push_dispatch_group(P, lr, gi, s_g0, s_g1, epoch);
    }
    __syncthreads();
    trace_mark(rv, 25);

    const int NCH = (H + kChunkCh - 1) / kChunkCh;
    // proxy transport: each block takes a contiguous range of (token, chunk)
    // items, so it touches few command groups and reports to each of them once
    const int n_items = T * NCH, ipb = (n_items + gridDim.x - 1) / gridDim.x;
    const int it0 = P.use_proxy ? blockIdx.x * ipb + warp : blockIdx.x * nw + warp;
    const int it_end = P.use_proxy ? min(n_items, (int)(blockIdx.x + 1) * ipb) : n_items;
    const int it_step = P.use_proxy ? nw : total_w;
    for (int item = it0; item < it_end; item += it_step) {
      const int t = item / NCH, ch = item % NCH;
      // the token's HBM loads first, so their latency overlaps the slot math
      const int ch0 = ch * kChunkCh + lane * 16;
      const bool active = ch0 < H;
      const int4* src = reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + (size_t)t * H * 2);
      int4 x0 = make_int4(0, 0, 0, 0), x1 = x0;
      if (active) {
        x0 = ld_nc_v4(src + ch0 / 8);
        x1 = ld_nc_v4(src + ch0 / 8 + 1);
      }
      uint64_t p = 0;
      int gid = -1;  // proxy: the command group of this lane's row
      if (lane < k) {
        const int e = s_e[t * k + lane];
        int32_t slot = -1;
        if (e >= 0) {
          const int d = e / L;
          if (P.use_proxy) {
            int loc = s_loc[t * k + lane];
            const bool dup = loc < -1;  // same expert twice in the token's top-k: one row
            if (dup) loc = s_loc[t * k + (-2 - loc)];
            const int row = rs[d * (T + 1) + t] + loc;
            if (!dup) {  // rows for a peer: my send block; rows for me: my receive block
              const int64_t blk = d == me ? g.off_disp_recv + (int64_t)(par * R + me) * g.disp_block
                                          : g.off_disp_send + (int64_t)(par * R + d) * g.disp_block;
              p = reinterpret_cast<uint64_t>(my_ll + blk + g.hdr_bytes + (int64_t)row * rstride);
              gid = group_of_row(s_g1, G, R, d, row);
            }
            slot = (int32_t)(d * g.rows_per_src + row);
          } else {
            const int row = pre[e] + ordinal_of(bm + (size_t)e * W, t);
            char* blk = rv.peer[d] + P.ll_off + g.off_disp_recv + (int64_t)(par * R + me) * g.disp_block;
            p = reinterpret_cast<uint64_t>(blk + g.hdr_bytes + (int64_t)row * rstride);
            slot = (int32_t)(d * g.rows_per_src + row);
          }
        }
        if (ch == 0) a.comb_slot[(size_t)t * k + lane] = slot;
      }
      if (g.use_fp8) {
        int4 q;
        const float sinv = quant16(x0, x1, active, a.round_scale, q);
        for (int j = 0; j < k; ++j) {
          char* pj = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, p, j));
          if (pj != nullptr && active) {
            st_v4(reinterpret_cast<int4*>(pj + ch0), q);
            if ((lane & 7) == 0) reinterpret_cast<float*>(pj + H)[ch0 / 128] = sinv;
          }
        }
      } else {
        for (int j = 0; j < k; ++j) {
          char* pj = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, p, j));
          if (pj != nullptr && active) {
            st_v4(reinterpret_cast<int4*>(pj + 2 * ch0), x0);
            st_v4(reinterpret_cast<int4*>(pj + 2 * ch0 + 16), x1);
          }
        }
      }
      if (ch == 0 && p != 0) {
        int32_t* meta = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(p) + meta_off);
        meta[0] = t;
        if (P.use_proxy) {  // token-major rows carry their expert and ordinal for the receiver
          const int e = s_e[t * k + lane];
          meta[1] = e % L;
          meta[2] = ordinal_of(bm + (size_t)e * W, t);
        }
      }
      if (P.use_proxy) {  // count this item's rows at their groups (block-local)
        const unsigned act = __ballot_sync(0xffffffffu, gid >= 0);
        if (gid >= 0) {
          const unsigned peers = __match_any_sync(act, gid);
          if (lane == __ffs(peers) - 1) atomicAdd(&s_arr[gid], (uint32_t)__popc(peers));
        }
      }
    }
    if (P.use_proxy) {
      // the block's rows are stored (bar.sync): report them to their groups,
      // one gpu-scope acq_rel add per touched group; the add that completes a
      // group pushes its WRITE at once — no grid-wide ticket on this path
      __syncthreads();
      trace_mark_max(rv, 36);  // the last block's rows are stored
      for (int gg = tid; gg < G; gg += blockDim.x) {
        const uint32_t n = s_arr[gg];
        if (n && atom_add_acq_rel_gpu(&sc->llp_grp[0][par][gg], n) + n == (uint32_t)s_gexp[gg])
          ll_push_dispatch_group(P, lr, gg, s_g0, s_g1, epoch);
      }
      // off the critical path: the send-block reuse rule held (one PCIe read)
      if (blockIdx.x == gridDim.x - 1 && tid >= 32 && tid - 32 < G) check_channel_backlog(rv, tid - 32, 2);
    }

    __shared__ uint32_t s_last;
    __syncthreads();
    trace_mark(rv, 26);
    if (!P.use_proxy) {
      // direct transport: every block signals every destination itself once its
      // rows are stored (release cumulativity over the block barrier); block 0
      // first writes each destination's per-expert count header.  No ticket,
      // no system fence on the receiver's critical path.
      if (blockIdx.x == 0) {
        for (int i = tid; i < R * L; i += blockDim.x) {
          const int d = i / L, le = i % L;
          char* blk = rv.peer[d] + P.ll_off + g.off_disp_recv + (int64_t)(par * R + me) * g.disp_block;
          reinterpret_cast<int32_t*>(blk)[le] = cnt[i];
        }
        __syncthreads();
      }
      if (tid < R) red_release_sys_add(&meta_of(rv.peer[tid])->ll_disp_cnt[par][me], 1u);
    }
    // the ticket only tracks the device-resident epoch (and, for the proxy
    // transport, hands the rows to the FIFO): the last block bumps it
    if (tid == 0) s_last = atom_add_acq_rel_gpu(&sc->ll_ticket[par], 1u) == gridDim.x - 1;
    __syncthreads();
    trace_mark(rv, 27);
    if (s_last && warp == 0) {
      for (int gg = lane; gg < kMaxFifo; gg += 32) sc->llp_grp[0][par][gg] = 0;
      if (lane == 0) {
        sc->ll_ticket[par] = 0;
        sc->ll_epoch[0] = epoch;
        if (P.use_proxy) sc->ll_pcnt[0] = base_pcnt + 1;
      }
    }
  }

  if (P.phases & 2) {
    // receive: wait for every source, then compact into the packed layout
    int32_t* s_hdr = reinterpret_cast<int32_t*>(smem);   // [R][L]
    int32_t* s_off = s_hdr + R * L;                       // [R][L] prefix over sources
    int32_t* s_pre = s_off + R * L;                       // [R][L] prefix over experts (row in block)
    int32_t* s_tot = s_pre + R * L;                       // [L + 1] prefix over experts of totals
    int32_t* s_rows = s_tot + L + 1;                      // [R + 1] proxy: prefix over sources of rows
    if (!P.use_proxy) {
      // cumulative: every call of this parity adds gridDim.x per source (the
      // grid width is pinned per context, epb_ll_dispatch)
      if (tid < R) wait_geq(rv, &my_meta->ll_disp_cnt[par][tid], ((epoch + 1u) >> 1) * gridDim.x, 0x600 + tid);
    } else {
      wait_proxy_recv(rv, my_meta, 0, P.ngroups, P.disp_channels, R, me, P.pthreads, P.chmap, pexp, 0x680,
                      P.poll_ns, P.poll_leader);
    }
    __syncthreads();
    trace_mark(rv, 28);
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
        s_pre[s * L + le] = s_hdr[s * L + le];
        run += s_hdr[s * L + le];
      }
      s_tot[le + 1] = run;
    }
    if (tid == 0) s_tot[0] = 0;
    __syncthreads();
    for (int s = warp; s <= R; s += nw) {
      if (s < R) warp_scan_smem(s_pre + s * L, L, lane, true);  // row of (s, le) inside block s
      else warp_scan_smem(s_tot + 1, L, lane, false);            // packed offset of expert le
    }
    if (P.use_proxy && tid == 0) {
      int run = 0;
      for (int s = 0; s < R; ++s) {
        s_rows[s] = run;
        for (int le = 0; le < L; ++le) run += s_hdr[s * L + le];
      }
      s_rows[R] = run;
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
    const int pay16 = g.use_fp8 ? H / 16 : H / 8;
    for (int item = blockIdx.x * nw + warp; item < N; item += total_w) {
      int le, j, s = 0, row;
      if (P.use_proxy) {
        // token-major rows: item = (source, row); the row's header names its
        // expert and its ordinal among the source's tokens for that expert
        while (s < R - 1 && item >= s_rows[s + 1]) ++s;
        row = item - s_rows[s];
        const int32_t* mp = reinterpret_cast<const int32_t*>(my_ll + g.off_disp_recv +
                                                             (int64_t)(par * R + s) * g.disp_block + g.hdr_bytes +
                                                             (int64_t)row * rstride + meta_off);
        int v = 0;
        if (lane < 2) v = __ldcg(mp + 1 + lane);
        le = __shfl_sync(0xffffffffu, v, 0);
        j = s_off[s * L + le] + __shfl_sync(0xffffffffu, v, 1);
      } else {
        int lo = 0, hi = L;  // find le: s_tot[le] <= item < s_tot[le+1]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_tot[mid] <= item) lo = mid; else hi = mid;
        }
        le = lo;
        j = item - s_tot[le];
        while (s < R - 1 && j >= s_off[s * L + le] + s_hdr[s * L + le]) ++s;
        row = s_pre[s * L + le] + (j - s_off[s * L + le]);
      }
      const char* rp = my_ll + g.off_disp_recv + (int64_t)(par * R + s) * g.disp_block + g.hdr_bytes + row * rstride;
      int4* dst = reinterpret_cast<int4*>(static_cast<char*>(a.packed_recv_x) +
                                          ((int64_t)le * RT + j) * (g.use_fp8 ? H : 2 * H));
      warp_copy<false>(reinterpret_cast<const int4*>(rp), dst, pay16, lane);
      if (g.use_fp8 && a.packed_recv_x_scales != nullptr)
        for (int q = lane; q < S; q += 32)
          a.packed_recv_x_scales[((int64_t)le * S + q) * RT + j] = __ldcg(reinterpret_cast<const float*>(rp + H) + q);
      if (lane == 0) {
        a.packed_recv_src_info[(int64_t)le * RT + j] = __ldcg(reinterpret_cast<const int32_t*>(rp + meta_off));
        a.recv_route[(int64_t)le * RT + j] = (int32_t)(s * g.rows_per_src + row);
      }
    }
    trace_mark_max(rv, 29);
  }
}

// ---------------------------------------------------------------------------
// LL combine
// ---------------------------------------------------------------------------
struct LLCombineParams {
  int n_local, phases, use_proxy, disp_channels, pthreads;
  int ngroups;
  int poll_ns, poll_leader;
  int chmap;
  RankView rv[kMaxLocal];
  epb_ll_combine_args_t a[kMaxLocal];
  LLGeom g;
  int64_t ll_off;
};

// The lane whose arrival completed combine group gid (source s = gid % R,
// chunk gid / R of the rows s sent me): one WRITE of those rows back into s's
// combine block, piggybacked signal, on FIFO channel disp_channels + gid.
__device__ __noinline__ void ll_push_combine_group(const LLCombineParams& P, int lr, int gid, const int32_t* s_g0,
                                                   const int32_t* s_g1, uint32_t epoch) {
  const RankView& rv = P.rv[lr];
  const LLGeom& g = P.g;
  const int R = g.R, me = rv.rank, par = epoch & 1, ch = P.disp_channels + gid;
  const int s = gid % R;
  Scratch* sc = scratch_of(rv.base);
  if (s == me) {  // rows returned to myself were stored into my receive block directly
    red_release_gpu_add(&sc->llp_self[1], 1u);
    return;
  }
  trace_mark_max_any(rv, 60);  // (ordering: fifo_push's cumulative release, see the dispatch)
  trace_mark_max_any(rv, 61);
  const int64_t rel = P.ll_off - (int64_t)kRegionHeader;
  const int64_t first = (int64_t)s_g0[gid] * g.comb_row;
  const int64_t src = rel + g.off_comb_send + (int64_t)(par * R + s) * g.comb_block + first;
  const int64_t dst = rel + g.off_comb_recv + (int64_t)(par * R + me) * g.comb_block + first;
  uint64_t lo, hi;
  cmd_pack_dev(EPB_CMD_WRITE, s, ch, src, dst, (int64_t)(s_g1[gid] - s_g0[gid]) * g.comb_row,
               EPB_FLAG_PIGGYBACK_ATOMIC, lo, hi);
  fifo_push(rv, ch, lo, hi);
  if (rv.trace && gid < 12) scratch_of(rv.base)->trace[52 + gid] = (int64_t)globaltimer();
}

__global__ void __launch_bounds__(kLLThreads, 1) ll_combine_kernel(const __grid_constant__ LLCombineParams P) {
  const int lr = blockIdx.y;
  const RankView& rv = P.rv[lr];
  const epb_ll_combine_args_t& a = P.a[lr];
  const LLGeom& g = P.g;
  const int R = g.R, L = g.L, H = g.H, me = rv.rank, k = g.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const int total_w = gridDim.x * nw;
  char* my_ll = rv.base + P.ll_off;
  Scratch* sc = scratch_of(rv.base);
  Meta* my_meta = meta_of(rv.base);
  const uint32_t base_epoch = *reinterpret_cast<volatile uint32_t*>(&sc->ll_epoch[1]);
  const uint32_t base_pcnt = *reinterpret_cast<volatile uint32_t*>(&sc->ll_pcnt[1]);
  const bool sending = (P.phases & 1) != 0;
  const uint32_t epoch = sending ? base_epoch + 1 : base_epoch;
  const uint64_t pexp = base_pcnt + ((sending && P.use_proxy) ? 1 : 0);
  const int par = epoch & 1;
  const int RT = R * g.Tmax;
  const int n16 = H / 8;
  __shared__ int32_t s_tot[kMaxLocalExperts + 1];
  trace_mark(rv, 32);

  if (sending) {
    for (int le = tid; le < L; le += blockDim.x) s_tot[le + 1] = a.packed_recv_count[le];
    if (tid == 0) s_tot[0] = 0;
    // proxy transport: rows each source sent me (= rows of its combine block),
    // split into command groups like the dispatch's
    __shared__ int32_t s_g0[kMaxFifo], s_g1[kMaxFifo], s_ns[kMaxRanks];
    __shared__ uint32_t s_arr[kMaxFifo];
    const int G = P.ngroups;
    for (int gg = tid; gg < G; gg += blockDim.x) s_arr[gg] = 0;
    if (P.use_proxy) {

      for (int src = tid; src < R; src += blockDim.x) {
        int n = 0;
        for (int le = 0; le < L; ++le) n += (int)(a.packed_recv_layout_range[le * R + src] & 0xffffffffll);
        s_ns[src] = n;
      }
    }
    __syncthreads();
    if (warp == 0) warp_scan_smem(s_tot + 1, L, lane, false);
    if (P.use_proxy) {
      for (int gg = tid; gg < G; gg += blockDim.x) {
        const int src = gg % R, c = gg / R, nc = group_chunks(G, R, src), n = s_ns[src];
        s_g0[gg] = (int)((int64_t)c * n / nc);
        s_g1[gg] = (int)((int64_t)(c + 1) * n / nc);
      }
      __syncthreads();
      if (blockIdx.x == 0)  // empty groups still signal once per call
        for (int gg = tid; gg < G; gg += blockDim.x)
          if (s_g1[gg] == s_g0[gg]) ll_push_combine_group(P, lr, gg, s_g0, s_g1, epoch);
    }
    __syncthreads();
    const int N = s_tot[L];
    const int ipb = (N + gridDim.x - 1) / gridDim.x;  // proxy: contiguous item range per block
    const int it0 = P.use_proxy ? blockIdx.x * ipb + warp : blockIdx.x * nw + warp;
    const int it_end = P.use_proxy ? min(N, (int)(blockIdx.x + 1) * ipb) : N;
    const int it_step = P.use_proxy ? nw : total_w;
    for (int item = it0; item < it_end; item += it_step) {
      int lo = 0, hi = L;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_tot[mid] <= item) lo = mid; else hi = mid;
      }
      const int le = lo, j = item - s_tot[le];
      const int route = a.recv_route[(int64_t)le * RT + j];
      const int s = (int)(route / g.rows_per_src), row = (int)(route % g.rows_per_src);
      char* blk = !P.use_proxy ? rv.peer[s] + P.ll_off + g.off_comb_recv + (int64_t)(par * R + me) * g.comb_block
                  : s == me    ? my_ll + g.off_comb_recv + (int64_t)(par * R + me) * g.comb_block
                               : my_ll + g.off_comb_send + (int64_t)(par * R + s) * g.comb_block;
      warp_copy<true>(reinterpret_cast<const int4*>(static_cast<const char*>(a.x) + ((int64_t)le * RT + j) * 2 * H),
                      reinterpret_cast<int4*>(blk + (int64_t)row * g.comb_row), n16, lane);
      if (P.use_proxy && lane == 0) atomicAdd(&s_arr[group_of_row(s_g1, G, R, s, row)], 1u);
    }
    if (P.use_proxy) {  // report the block's rows to their groups (see the dispatch)
      __syncthreads();
      trace_mark_max(rv, 37);
      for (int gg = tid; gg < G; gg += blockDim.x) {
        const uint32_t n = s_arr[gg];
        if (n && atom_add_acq_rel_gpu(&sc->llp_grp[1][par][gg], n) + n == (uint32_t)(s_g1[gg] - s_g0[gg]))
          ll_push_combine_group(P, lr, gg, s_g0, s_g1, epoch);
      }
      if (blockIdx.x == gridDim.x - 1 && tid >= 32 && tid - 32 < G) check_channel_backlog(rv, P.disp_channels + tid - 32, 2);
    }
    __shared__ uint32_t s_last;
    __syncthreads();
    trace_mark(rv, 33);
    if (!P.use_proxy && tid < R) red_release_sys_add(&meta_of(rv.peer[tid])->ll_comb_cnt[par][me], 1u);
    if (tid == 0) s_last = atom_add_acq_rel_gpu(&sc->ll_ticket[2 + par], 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last && warp == 0) {
      for (int gg = lane; gg < kMaxFifo; gg += 32) sc->llp_grp[1][par][gg] = 0;
      if (lane == 0) {
        sc->ll_ticket[2 + par] = 0;
        sc->ll_epoch[1] = epoch;
        if (P.use_proxy) sc->ll_pcnt[1] = base_pcnt + 1;
      }
    }
  }

  if (P.phases & 2) {
    const int T = a.num_tokens;
    const int NCC = (n16 + 63) / 64;  // 64 x 16 B columns per item (2 per lane)
    // each warp's first two items: their routing slots and weights are loaded
    // before the wait for the peers, off the critical path
    int pre_slot[2] = {-1, -1};
    float pre_w[2] = {0.0f, 0.0f};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int item = blockIdx.x * nw + warp + q * total_w;
      if (item < T * NCC && lane < k) {
        const int t = item / NCC;
        pre_slot[q] = a.comb_slot[(size_t)t * k + lane];
        pre_w[q] = a.topk_weights[(size_t)t * k + lane];
      }
    }
    if (!P.use_proxy) {
      if (tid < R) wait_geq(rv, &my_meta->ll_comb_cnt[par][tid], ((epoch + 1u) >> 1) * gridDim.x, 0x700 + tid);
    } else {
      wait_proxy_recv(rv, my_meta, 1, P.ngroups, P.disp_channels, R, me, P.pthreads, P.chmap, pexp, 0x780,
                      P.poll_ns, P.poll_leader);
    }
    __syncthreads();
    trace_mark(rv, 34);
    const char* recv = my_ll + g.off_comb_recv + (int64_t)par * R * g.comb_block;
    int q = 0;
    for (int item = blockIdx.x * nw + warp; item < T * NCC; item += total_w, ++q) {
      const int t = item / NCC, i0 = (item % NCC) * 64 + lane, i1 = i0 + 32;
      uint64_t p = 0;
      float w = 0.0f;
      if (lane < k) {
        const int slot = q < 2 ? pre_slot[q] : a.comb_slot[(size_t)t * k + lane];
        if (slot >= 0) {
          const int r = (int)(slot / g.rows_per_src), row = (int)(slot % g.rows_per_src);
          p = reinterpret_cast<uint64_t>(recv + (int64_t)r * g.comb_block + (int64_t)row * g.comb_row);
          w = q < 2 ? pre_w[q] : a.topk_weights[(size_t)t * k + lane];
        }
      }
      float acc0[8], acc1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc0[q] = acc1[q] = 0.0f;
      for (int jg = 0; jg < k; jg += 8) {
        int4 v0[8], v1[8];
        float wj[8];
        bool ok[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = min(jg + jj, 31);
          const uint64_t pj = __shfl_sync(0xffffffffu, p, j);
          wj[jj] = __shfl_sync(0xffffffffu, w, j);
          ok[jj] = (jg + jj < k) && pj != 0;
          const int4* rp = reinterpret_cast<const int4*>(pj);
          if (ok[jj] && i0 < n16) v0[jj] = ld_cg_v4(rp + i0);
          if (ok[jj] && i1 < n16) v1[jj] = ld_cg_v4(rp + i1);
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          if (!ok[jj]) continue;
          const uint32_t u0[4] = {(uint32_t)v0[jj].x, (uint32_t)v0[jj].y, (uint32_t)v0[jj].z, (uint32_t)v0[jj].w};
          const uint32_t u1[4] = {(uint32_t)v1[jj].x, (uint32_t)v1[jj].y, (uint32_t)v1[jj].z, (uint32_t)v1[jj].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (i0 < n16) {
              acc0[2 * q] = __fadd_rn(acc0[2 * q], __fmul_rn(wj[jj], bf16lo(u0[q])));
              acc0[2 * q + 1] = __fadd_rn(acc0[2 * q + 1], __fmul_rn(wj[jj], bf16hi(u0[q])));
            }
            if (i1 < n16) {
              acc1[2 * q] = __fadd_rn(acc1[2 * q], __fmul_rn(wj[jj], bf16lo(u1[q])));
              acc1[2 * q + 1] = __fadd_rn(acc1[2 * q + 1], __fmul_rn(wj[jj], bf16hi(u1[q])));
            }
          }
        }
      }
      int4* out = reinterpret_cast<int4*>(static_cast<char*>(a.combined_x) + (size_t)t * H * 2);
      uint32_t o[4];
      if (i0 < n16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __nv_bfloat162 h = __floats2bfloat162_rn(acc0[2 * q], acc0[2 * q + 1]);
          o[q] = *reinterpret_cast<uint32_t*>(&h);
        }
        st_na_v4(out + i0, make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]));
      }
      if (i1 < n16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __nv_bfloat162 h = __floats2bfloat162_rn(acc1[2 * q], acc1[2 * q + 1]);
          o[q] = *reinterpret_cast<uint32_t*>(&h);
        }
        st_na_v4(out + i1, make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]));
      }
    }
    trace_mark_max(rv, 35);
  }
}

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
  if (c->cfg.fifo_channels > 0 && c->ll_off() - kRegionHeader + c->cfg.ll_bytes > 0xFFFFFFFFull)
    return epb_set_error(EPB_ERR_CONFIG, "proxy transport: 32-bit TransferCmd offsets need "
                                         "num_nvl_bytes + num_rdma_bytes < 4 GiB");
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

// The direct transport's completion counters are cumulative per source (each
// call adds one per sender block), so a context keeps the grid width of its
// first call of each kind; every rank derives the same width from the same
// num_sms.  Returns 0 if that width can no longer be co-resident.
static int ll_blocks(epb_t* const* ctxs, int n_local, int num_sms, const void* kernel, size_t smem, int kind) {
  const int max_active = std::max(1, epb_max_active_blocks(kernel, kLLThreads, smem));
  const int cap = std::max(1, max_active * ctxs[0]->num_sms / n_local);
  int& pinned = ctxs[0]->ll_grid[kind];
  if (pinned == 0) pinned = std::min(std::max(1, num_sms / n_local), cap);
  for (int i = 1; i < n_local; ++i) ctxs[i]->ll_grid[kind] = pinned;
  return pinned <= cap ? pinned : 0;
}

// Command groups per destination rank for the proxy transport (EPB_LL_GROUPS_PER_RANK,
// default 1): each group is one WRITE the proxy turns into one cudaMemcpyAsync, which
// costs the host 3-6 us (profiles/r02_ll_proxy.md), so finer groups only pay when the
// copies are large enough to overlap that cost.
// Receive polling of the proxy transport: EPB_LL_POLL_NS (sleep between polls,
// default 200 ns), EPB_LL_POLL_LEADER=1 (block 0 alone polls the signal words).
static void ll_poll(int* ns, int* leader) {
  static const int v_ns = [] {
    const char* s = std::getenv("EPB_LL_POLL_NS");
    return s ? std::max(0, std::atoi(s)) : 200;
  }();
  static const int v_leader = [] {
    const char* s = std::getenv("EPB_LL_POLL_LEADER");
    return s ? std::atoi(s) : 0;
  }();
  *ns = v_ns;
  *leader = v_leader;
}

static int ll_groups(int world, int disp_channels) {
  static const int per = [] {
    const char* s = std::getenv("EPB_LL_GROUPS_PER_RANK");
    return s ? std::max(1, std::atoi(s)) : 1;
  }();
  return world * std::max(1, std::min(per, disp_channels / std::max(1, world)));
}

static int ll_transport(epb_ctx* c, int use_proxy, int* disp_channels, int* pthreads) {
  *pthreads = 1;
  if (use_proxy) {
    if (c->cfg.fifo_channels < 2 || !c->proxy)
      return epb_set_error(EPB_ERR_UNSUPPORTED, "proxy transport needs >= 2 FIFO channels and a running proxy");
    *disp_channels = c->cfg.fifo_channels / 2;  // one command group per channel, dispatch and combine halves
    if (*disp_channels < c->world)
      return epb_set_error(EPB_ERR_CONFIG, "LL proxy transport needs fifo_channels >= 2 x world (a group per rank)");
    *pthreads = epb_proxy_nthreads(c);
  } else {
    *disp_channels = std::max(1, c->cfg.fifo_channels / 2);
  }
  return EPB_OK;
}

extern "C" int epb_ll_dispatch(epb_t* const* ctxs, int n_local, const epb_ll_dispatch_args_t* args, int num_sms,
                               void* stream) {
  if (int e = check_group_ll(ctxs, n_local)) return e;
  LLDispatchParams P;
  std::memset(&P, 0, sizeof(P));
  const epb_ll_dispatch_args_t& a0 = args[0];
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
    if (int e = ll_transport(c, P.use_proxy, &P.disp_channels, &P.pthreads)) return e;
    P.ngroups = ll_groups(c->world, P.disp_channels);
    ll_poll(&P.poll_ns, &P.poll_leader);
    P.chmap = c->proxy_chmap;
    P.rv[i] = c->view();
    P.a[i] = args[i];
  }
  const int W = std::max(1, (a0.max_tokens + 31) / 32);
  size_t smem_send = ((size_t)P.g.E * W + 2 * P.g.E) * 4 + (size_t)a0.max_tokens * a0.num_topk * 2;
  if (P.use_proxy)  // token-major slots [T][k] int16 + first row per (destination, token)
    smem_send += (size_t)a0.max_tokens * a0.num_topk * 2 + (size_t)P.g.R * (a0.max_tokens + 1) * 4;
  const size_t smem_recv = (size_t)(3 * P.g.R * P.g.L + P.g.L + 1 + P.g.R + 1) * 4;
  const size_t smem = std::max(smem_send, smem_recv);
  if (smem > 200 * 1024) return epb_set_error(EPB_ERR_CONFIG, "LL dispatch shape needs too much shared memory");
  epb_set_carveout((const void*)ll_dispatch_kernel);
  EPB_CUDA(epb_ensure_smem((const void*)ll_dispatch_kernel, smem));
  const int nb = ll_blocks(ctxs, n_local, num_sms, (const void*)ll_dispatch_kernel, smem, 0);
  if (nb == 0) return epb_set_error(EPB_ERR_CONFIG, "LL dispatch: this shape no longer fits the context's pinned grid");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(epb_launch_grid_sync((void*)ll_dispatch_kernel, dim3(nb, n_local), dim3(kLLThreads), kargs, smem, st));
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
    if (int e = ll_transport(c, P.use_proxy, &P.disp_channels, &P.pthreads)) return e;
    P.ngroups = ll_groups(c->world, P.disp_channels);
    ll_poll(&P.poll_ns, &P.poll_leader);
    P.chmap = c->proxy_chmap;
    P.rv[i] = c->view();
    P.a[i] = args[i];
  }
  epb_set_carveout((const void*)ll_combine_kernel);  // same split as ll_dispatch_kernel
  const int nb = ll_blocks(ctxs, n_local, num_sms, (const void*)ll_combine_kernel, 0, 1);
  if (nb == 0) return epb_set_error(EPB_ERR_CONFIG, "LL combine: grid no longer co-resident");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* kargs[] = {&P};
  EPB_CUDA(epb_launch_grid_sync((void*)ll_combine_kernel, dim3(nb, n_local), dim3(kLLThreads), kargs, 0, st));
  return EPB_OK;
}

extern "C" int epb_per_token_cast_to_fp8(const void* x, int num_tokens, int hidden, int round_scale, void* q,
                                         float* scales, void* stream) {
  if (hidden <= 0 || hidden % 128) return epb_set_error(EPB_ERR_CONFIG, "hidden must be a multiple of 128");
  if (num_tokens <= 0) return EPB_OK;
  const int warps_per_block = kLLThreads / 32;
  const int items = num_tokens * ((hidden + kChunkCh - 1) / kChunkCh);
  const int blocks = std::min(148 * 8, (items + warps_per_block - 1) / warps_per_block);
  fp8_cast_kernel<<<blocks, kLLThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), num_tokens, hidden, round_scale, static_cast<uint8_t*>(q), scales);
  EPB_CUDA(cudaGetLastError());
  return EPB_OK;
}

// Load this file's kernels now (see epb_preload_kernels, api.cpp).
cudaError_t epb_preload_ll() {
  cudaFuncAttributes attr;
  for (const void* fn : {(const void*)fp8_cast_kernel, (const void*)ll_dispatch_kernel, (const void*)ll_combine_kernel})
    if (cudaError_t e = cudaFuncGetAttributes(&attr, fn)) return e;
  return cudaSuccess;
}
