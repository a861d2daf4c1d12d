/*
 * epb.h — C ABI of the B200-native expert-parallel dispatch/combine path.
 *
 * This is the drop-in boundary (libepb200.so).  Every entry point takes plain
 * pointers, sizes and a `void* stream` (a cudaStream_t); no torch types cross
 * it.  Device pointers are raw CUDA device addresses; "host" pointers are
 * plain host memory.  Every function returns an EPB_* code (0 = ok) and
 * records a message retrievable with epb_last_error().
 *
 * The reference (/root/reference/pkg/src/epsim) has no FFI of its own: its
 * callable surface is Python functions over numpy arrays, and the DeepEP API
 * it claims compatibility with is external.  Each
 * declaration below cites the reference interface (file:line) or the
 * DeepEP-style API method it replaces.  See INTEGRATION.md for the ctypes
 * binding the Python host layer uses.
 */
#ifndef EPB_H_
#define EPB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Static limits of one NVLink domain (one HGX B200 node). */
#define EPB_MAX_RANKS 8
#define EPB_MAX_LOCAL 8 /* ranks emulated inside one process (test harness) */
#define EPB_MAX_CHANNELS 256
#define EPB_MAX_LOCAL_EXPERTS 1024
#define EPB_IPC_HANDLE_BYTES 64

/* Error codes, 1:1 with the exception classes of errors.py:4-43. */
enum {
  EPB_OK = 0,
  EPB_ERR_PROTOCOL = 1,    /* ProtocolViolation   errors.py:8  */
  EPB_ERR_SHUTDOWN = 2,    /* ChannelShutdown     errors.py:12 */
  EPB_ERR_CONFIG = 3,      /* ConfigError         errors.py:16 */
  EPB_ERR_FAULT = 4,       /* FaultError          errors.py:20 */
  EPB_ERR_CONNECTION = 5,  /* ConnectionError_    errors.py:30 */
  EPB_ERR_UNSUPPORTED = 6, /* UnsupportedOperation errors.py:34 */
  EPB_ERR_INVARIANT = 7,   /* InvariantViolation  errors.py:38 */
  EPB_ERR_DEADLOCK = 8,    /* RingDeadlock        errors.py:42 */
  EPB_ERR_CUDA = 9         /* CUDA runtime failure (no reference analogue) */
};

/* TransferCmd kinds / flags (command.py:25-34) and imm kinds (imm.py:20-23). */
enum { EPB_CMD_WRITE = 0, EPB_CMD_ATOMIC = 1, EPB_CMD_DRAIN = 2, EPB_CMD_BARRIER = 3 };
enum { EPB_FLAG_PIGGYBACK_ATOMIC = 1, EPB_FLAG_SAME_RAIL_BARRIER = 2 };

/* SPSC ring control-array layout, identical to kernels.py:23-31 (int64 word
 * indices; counters a cache line apart; slots of 2 words follow). */
enum { EPB_CTL_TAIL = 0, EPB_CTL_HEAD = 8, EPB_CTL_COMPLETED = 16, EPB_CTL_FLAGS = 24, EPB_CTL_SLOT0 = 32 };
enum { EPB_RING_FLAG_SHUTDOWN = 1 };

typedef struct epb_ctx epb_t;

/* ------------------------------------------------------------------------ */
/* Context / bootstrap  (replaces SPEC.md:244-252 proxy.start + the         */
/* symmetric-region handshake SPEC.md:237-241; DeepEP Buffer.__init__).      */
/* ------------------------------------------------------------------------ */
typedef struct {
  size_t nvl_bytes;     /* normal-mode arena: recv slots + combine staging */
  size_t ll_bytes;      /* low-latency region (0 = LL disabled)             */
  int num_recv_slots;   /* dispatch receive slots carved from nvl_bytes      */
  int fifo_channels;    /* GPU->CPU command FIFOs (0 = no proxy)            */
  int fifo_capacity;    /* kMaxInflight per FIFO, power of two */
  int proxy_threads;    /* CPU proxy threads (PAPER.md:469 uses 4)          */
  int ht_transport;     /* normal mode data path (EPB_HT_*): NVLink stores from
                           the kernels into worst-case receive slots; the CPU
                           proxy (WRITE/ATOMIC TransferCmds; the arena then also
                           holds one send-staging slot); or bounded chunked
                           ring channels (the arena holds only the rings)    */
} epb_config_t;

enum { EPB_HT_NVLINK = 0, EPB_HT_PROXY = 1, EPB_HT_RING = 2 };

int epb_create(epb_t** out, int rank, int world, const epb_config_t* cfg);
int epb_destroy(epb_t* ctx);
/* cudaIpcMemHandle_t bytes of this rank's symmetric region. */
int epb_ipc_handle(epb_t* ctx, void* out_handle /* EPB_IPC_HANDLE_BYTES */);
/* Map every peer's region (handles: world x EPB_IPC_HANDLE_BYTES, own entry ignored). */
int epb_open_peers(epb_t* ctx, const void* handles);
/* Test harness: treat n contexts living in this process as ranks 0..n-1 of one group. */
int epb_link_local(epb_t* const* ctxs, int n);
const char* epb_last_error(void);
/* Device-reported error word (set by kernels on spin timeout / capacity overflow). */
int epb_device_error(epb_t* ctx, int64_t* detail);
int epb_clear_device_error(epb_t* ctx);
int epb_num_sms(void);
/* Phase timestamps (64 x %globaltimer ns) recorded by the kernels when EPB_TRACE=1. */
int epb_trace(epb_t* ctx, int64_t* out64);
/* Diagnostics: one thread writes %globaltimer (ns) to the device word *dst, in
   stream order (brackets launches on the same clock as epb_trace's marks). */
int epb_debug_stamp(int64_t* dst, void* stream);
/* Diagnostics: LL proxy device state (16 int64: llp_self[2], ll_pcnt[2], ll_epoch[2],
   llp_grp[0][0..4], llp_grp[1][0..4]). */
int epb_debug_ll_state(epb_t* ctx, int64_t* out16);
/* Diagnostics: byte offset of the proxy HT signal counters in a region. */
int64_t epb_debug_ht_sig_offset(void);
/* Byte offset of the arena inside a region (TransferCmd offsets are relative to it). */
int64_t epb_arena_offset(void);
/* Base device address of this rank's symmetric region and its size. */
int epb_region(epb_t* ctx, void** base, size_t* bytes);

/* ------------------------------------------------------------------------ */
/* Layout  (DeepEP Buffer.get_dispatch_layout; SPEC.md:416-424 plan_dedup)   */
/* ------------------------------------------------------------------------ */
int epb_get_dispatch_layout(const int64_t* topk_idx, int num_tokens, int num_topk, int num_experts,
                            int num_ranks, int32_t* num_tokens_per_rank, int32_t* num_tokens_per_expert,
                            uint8_t* is_token_in_rank, void* stream);

/* ------------------------------------------------------------------------ */
/* Normal (high-throughput) mode  (DeepEP Buffer.dispatch / Buffer.combine;  */
/* SPEC.md:436-454 dispatch_ht / combine)                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t cap_rows;        /* rows a recv slot / combine staging holds          */
  int64_t slot_bytes;      /* bytes per recv slot                               */
  int64_t off_x, off_scales, off_topk_idx, off_topk_w, off_src_idx; /* within a slot */
  int64_t comb_off[2];     /* combine staging (parity) offsets in the region     */
  int64_t comb_w_off;      /* weights offset inside a combine staging buffer     */
  int64_t slot0_off;       /* offset of slot 0 in the region                     */
  int64_t send_off;        /* proxy transport: send-staging slot offset (else 0) */
  int64_t comb_flag_off;   /* per-row arrival words inside a combine staging buffer
                              (streamed push combine: the call epoch, stored after
                              the row)                                             */
} epb_recv_layout_t;

int epb_recv_layout(epb_t* ctx, int hidden, int num_topk, epb_recv_layout_t* out);

typedef struct {
  /* inputs */
  const void* x;              /* [T, hidden] bf16 (elem_bytes 2) or e4m3 (1)   */
  const float* x_scales;      /* [T, num_scales] f32 or NULL                   */
  int hidden, elem_bytes, num_scales;
  const int64_t* topk_idx;    /* [T, num_topk] or NULL                         */
  const float* topk_weights;  /* [T, num_topk] or NULL                         */
  int num_topk;
  const uint8_t* is_token_in_rank;       /* [T, R] bool                         */
  const int32_t* num_tokens_per_expert;  /* [E] or NULL (cached handle)         */
  int num_tokens, num_experts, expert_alignment;
  int recv_slot;              /* arena slot this rank receives into            */
  /* handle outputs */
  int32_t* rank_prefix_matrix;         /* [R, R]  inclusive over source rank    */
  int32_t* channel_prefix_matrix;      /* [R, C]  my sends, inclusive over chan */
  int32_t* recv_channel_prefix_matrix; /* [R, C]  my receives, inclusive        */
  int32_t* send_head;                  /* [T, R]  row of t inside my block at r, -1 */
  /* DeepEP num_worst_tokens: > 0 = the caller sized its receive views for this
     many rows and does not wait for the counts (no host sync, CUDA-graph
     capturable); rows [N_recv, num_worst_tokens) get recv_topk_idx = -1 and a
     call receiving more rows aborts with EPB_ERR_CONFIG */
  int num_worst_tokens;
} epb_dispatch_args_t;

/* One cooperative launch: per-channel counts, the cross-rank count exchange
 * (one NVLink mailbox round trip), prefix sums, then every deduplicated row
 * pushed straight into its final row of the destination's receive slot. */
int epb_dispatch(epb_t* const* ctxs, int n_local, const epb_dispatch_args_t* args, int num_channels,
                 void* stream);
/* Host wait for the receive counts the dispatch kernel publishes to pinned
 * memory mid-kernel.  per_expert: [num_local_experts] or NULL. */
int epb_wait_notify(epb_t* ctx, int64_t* num_recv, int32_t* num_recv_per_expert, int num_local_experts,
                    double timeout_s);

typedef struct {
  const void* x;              /* [N_recv, hidden] bf16, my receive order        */
  const float* topk_weights;  /* [N_recv, num_topk] or NULL                     */
  int num_recv, hidden, num_topk;
  const int32_t* rank_prefix_matrix;
  const uint8_t* is_token_in_rank;
  const int32_t* send_head;
  const int32_t* channel_prefix_matrix;       /* [R, C] from the dispatch handle */
  const int32_t* recv_channel_prefix_matrix;  /* [R, C] from the dispatch handle */
  int num_channels;                           /* C of the dispatch (combine grid) */
  int num_tokens;
  void* combined_x;              /* [T, hidden] bf16                            */
  float* combined_topk_weights;  /* [T, num_topk] or NULL                       */
} epb_combine_args_t;

int epb_combine(epb_t* const* ctxs, int n_local, const epb_combine_args_t* args, int num_sms, void* stream);

/* ------------------------------------------------------------------------ */
/* Chunked ring channels (SPEC.md:409-413 RingChannel,        */
/* :436-444 dispatch_ht; imm.py:28-31 HT_ROLE_HEAD credit   */
/* return).  ht_transport = EPB_HT_RING: the arena holds only bounded rings,   */
/* one per (source rank, lane) at every receiver for the dispatch and one per  */
/* (expert rank, lane) at every source for the combine; the receive tensors    */
/* are ordinary device memory sized from the notified counts.  A sender        */
/* writes 32-token chunks into the ring slots tail..tail+n,      */
/* then release-stores the tail; the receiver copies (dispatch) or reduces      */
/* (combine) them and release-stores the head back at the sender (credit).     */
/* ------------------------------------------------------------------------ */
typedef struct {
  int lanes;              /* ring lanes (sender + receiver block pair each)      */
  int ring_tokens;        /* slots per ring, a multiple of the 32-token chunk     */
  int64_t disp_slot_bytes, comb_slot_bytes;
  int64_t disp_off, comb_off;  /* ring areas inside the region                  */
  int64_t bytes_needed;
} epb_ring_layout_t;

/* Ring geometry for rows of `hidden` (bf16 sized) and num_topk; lanes <= 0
   picks the default for n_local ranks per GPU. */
int epb_ring_layout(epb_t* ctx, int hidden, int num_topk, int lanes, int n_local, epb_ring_layout_t* out);

/* The count exchange of epb_dispatch alone: fills the handle outputs
   (rank/channel prefix matrices, send_head) and publishes the host counts
   (epb_wait_notify); no rows move and no receive-slot capacity applies. */
int epb_dispatch_notify(epb_t* const* ctxs, int n_local, const epb_dispatch_args_t* args, int num_channels,
                        void* stream);

typedef struct {
  const void* x;              /* [T, hidden] bf16 (elem_bytes 2) or e4m3 (1)   */
  const float* x_scales;      /* [T, num_scales] or NULL                       */
  int hidden, elem_bytes, num_scales;
  const int64_t* topk_idx;    /* [T, num_topk] or NULL                         */
  const float* topk_weights;  /* [T, num_topk] or NULL                         */
  int num_topk, num_tokens, num_experts;
  const int32_t* rank_prefix_matrix;          /* from epb_dispatch_notify       */
  const int32_t* recv_channel_prefix_matrix;
  const int32_t* send_head;
  int num_channels;                           /* C of epb_dispatch_notify       */
  void* recv_x;               /* [N_recv, hidden] (device memory of the caller) */
  float* recv_x_scales;       /* [N_recv, num_scales] or NULL                  */
  int64_t* recv_topk_idx;     /* [N_recv, num_topk] or NULL                    */
  float* recv_topk_weights;   /* [N_recv, num_topk] or NULL                    */
  int32_t* recv_src_idx;      /* [N_recv]                                      */
  int num_recv;               /* N_recv (from epb_wait_notify): receive rows are
                                 bounds-checked against it                     */
} epb_ring_dispatch_args_t;

int epb_ring_dispatch(epb_t* const* ctxs, int n_local, const epb_ring_dispatch_args_t* args, int lanes,
                      void* stream);

typedef struct {
  const void* x;              /* [N_recv, hidden] bf16 expert outputs, my receive order */
  const float* topk_weights;  /* [N_recv, num_topk] or NULL                    */
  int num_recv, hidden, num_topk;
  const int32_t* rank_prefix_matrix;
  const int32_t* recv_channel_prefix_matrix;
  const int32_t* send_head;
  int num_channels;
  int num_tokens;
  void* combined_x;              /* [T, hidden] bf16                            */
  float* combined_topk_weights;  /* [T, num_topk] or NULL                       */
} epb_ring_combine_args_t;

int epb_ring_combine(epb_t* const* ctxs, int n_local, const epb_ring_combine_args_t* args, int lanes,
                     void* stream);

/* ------------------------------------------------------------------------ */
/* Low-latency mode  (DeepEP low_latency_dispatch/combine)  */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t rows_per_src;   /* rows one source block can hold (Tmax*min(k,L))   */
  int64_t disp_row_bytes; /* one dispatched message row                        */
  int64_t comb_row_bytes;
  int64_t bytes_needed;   /* LL region bytes needed for this shape            */
} epb_ll_layout_t;

int epb_ll_layout(int num_ranks, int max_tokens, int hidden, int num_topk, int num_experts, int use_fp8,
                  epb_ll_layout_t* out);

typedef struct {
  const void* x;              /* [T, hidden] bf16 */
  const int64_t* topk_idx;    /* [T, num_topk] */
  int num_tokens, num_topk, hidden, num_experts, max_tokens;
  int use_fp8, round_scale;
  void* packed_recv_x;                 /* [L, R*Tmax, hidden] e4m3 or bf16            */
  float* packed_recv_x_scales;         /* [L, hidden/128, R*Tmax] (token dim contiguous) */
  int32_t* packed_recv_count;          /* [L]                                         */
  int32_t* packed_recv_src_info;       /* [L, R*Tmax] source token index               */
  int64_t* packed_recv_layout_range;   /* [L, R]  (begin << 32) | count               */
  int32_t* recv_route;                 /* [L, R*Tmax] internal: row in source block    */
  int32_t* comb_slot;                  /* [T, num_topk] internal: row of (t,k) in my combine recv */
  int phases;                          /* 1 = send, 2 = receive, 3 = both             */
  int use_proxy;                       /* route the copies through the CPU proxy FIFO  */
} epb_ll_dispatch_args_t;

int epb_ll_dispatch(epb_t* const* ctxs, int n_local, const epb_ll_dispatch_args_t* args, int num_sms,
                    void* stream);

typedef struct {
  const void* x;                       /* [L, R*Tmax, hidden] bf16 expert outputs */
  const int64_t* topk_idx;             /* [T, num_topk] */
  const float* topk_weights;           /* [T, num_topk] */
  const int32_t* packed_recv_count;    /* [L] */
  const int64_t* packed_recv_layout_range; /* [L, R] */
  const int32_t* recv_route;           /* [L, R*Tmax] */
  const int32_t* comb_slot;            /* [T, num_topk] */
  int num_tokens, num_topk, hidden, num_experts, max_tokens;
  void* combined_x;                    /* [T, hidden] bf16 */
  int phases, use_proxy;
} epb_ll_combine_args_t;

int epb_ll_combine(epb_t* const* ctxs, int n_local, const epb_ll_combine_args_t* args, int num_sms,
                   void* stream);

/* FP8 e4m3 per-128-channel cast (the LL quantiser as a standalone op, for the
 * FP8 normal-mode config).  x [T, hidden] bf16 -> q [T, hidden] e4m3, scales [T, hidden/128]. */
int epb_per_token_cast_to_fp8(const void* x, int num_tokens, int hidden, int round_scale, void* q, float* scales,
                              void* stream);

/* ------------------------------------------------------------------------ */
/* TransferCmd codec  (command.py:70-158)                                    */
/* ------------------------------------------------------------------------ */
/* pack(): validates like TransferCmd.validate (command.py:55-67). */
int epb_cmd_pack(int64_t kind, int64_t dst_rank, int64_t channel_id, int64_t src_offset, int64_t dst_offset,
                 int64_t length_or_value, int64_t flags, uint64_t* lo, uint64_t* hi);
/* pack_fields(): no validation, like command.py:113-138. */
int epb_cmd_pack_fields(const int64_t* kind, const int64_t* dst_rank, const int64_t* channel_id,
                        const int64_t* src_offset, const int64_t* dst_offset, const int64_t* length_or_value,
                        const int64_t* flags, int64_t n, uint64_t* lo, uint64_t* hi);
/* unpack_fields(): rejects reserved bits like command.py:141-146. */
int epb_cmd_unpack_fields(const uint64_t* lo, const uint64_t* hi, int64_t n, int64_t* kind, int64_t* dst_rank,
                          int64_t* channel_id, int64_t* src_offset, int64_t* dst_offset, int64_t* length_or_value,
                          int64_t* flags);

/* Immediate words (imm.py:75-91). */
int epb_imm_encode_ll_batch(const int64_t* kind, const int64_t* counter_index, const int64_t* operand, int64_t n,
                            int64_t* out);
int epb_imm_encode_ht_batch(const int64_t* kind, const int64_t* channel_id, const int64_t* sequence,
                            const int64_t* operand, int64_t n, int64_t* out);

/* ------------------------------------------------------------------------ */
/* SPSC command ring over the kernels.py:23-31 control array                 */
/* (kernels.py:61-104 push_batch / pop_batch, with release/acquire per       */
/* SPEC.md:111 instead of the reference's plain stores).                     */
/* ------------------------------------------------------------------------ */
int64_t epb_ring_push_batch(int64_t* ctl, int64_t cap, const int64_t* lo, const int64_t* hi, int64_t start,
                            int64_t want, int64_t max_spin);
int64_t epb_ring_pop_batch(int64_t* ctl, int64_t cap, int64_t* lo_out, int64_t* hi_out, int64_t start,
                           int64_t want, int64_t max_spin);
/* FifoChannel.poll: head command without dequeueing; returns 1 if present, 0 if empty. */
int epb_ring_poll(const int64_t* ctl, int64_t cap, int64_t* lo, int64_t* hi);
/* FifoChannel.mark_completed: COMPLETED = max(COMPLETED, upto); upto > HEAD is a
 * ProtocolViolation.  COMPLETED counts completed commands: command idx is complete iff COMPLETED > idx. */
int epb_ring_mark_completed(int64_t* ctl, int64_t upto);
/* FifoChannel.check_completion: 1 if command idx has completed, else 0. */
int epb_ring_check_completion(const int64_t* ctl, int64_t idx);
/* Set FLAG_SHUTDOWN (kernels.py:30): later pushes return -EPB_ERR_SHUTDOWN. */
int epb_ring_shutdown(int64_t* ctl);

/* Receiver-side delivery application (kernels.py:124-318), C++ port. */
int epb_apply_deliveries(uint8_t* regions, int64_t ep, int64_t region_len, int64_t* counters, int64_t n_counters,
                         int64_t n_counters_used, int64_t counter_base, int64_t mode_ht, int64_t n,
                         const int64_t* t_del, const int64_t* src_rank, const int64_t* dst_rank,
                         const int64_t* src_off, const int64_t* dst_off, const int64_t* length, const int64_t* op_hw,
                         const int64_t* imm_arr, const int64_t* work_id, int64_t* ll_counts, int32_t* ll_pend_x,
                         int32_t* ll_pend_d, int32_t* ll_pend_n, int64_t pmax, int64_t* ht_applied,
                         int32_t* ht_pend, int64_t n_channels, int64_t wmax, int64_t* eff_t, int64_t* eff_kind,
                         int64_t* eff_dst, int64_t* eff_src, int64_t* eff_key, int64_t* eff_aux,
                         int64_t* eff_counter, int64_t* eff_work, int64_t eff_cap, int64_t* esc_idx,
                         int64_t esc_cap, int64_t* result4);
/* Extra error codes of the port beyond kernels.py:41-47 (ERR_OK..ERR_BAD_IMM_KIND = 0..6). */
enum { EPB_DLV_ERR_FAULT = 7, EPB_DLV_ERR_EFFECT_OVERFLOW = 8 };

/* ------------------------------------------------------------------------ */
/* GPU -> CPU command FIFO + proxy        */
/* ------------------------------------------------------------------------ */
/* Pinned, device-mapped control array of FIFO `channel` (kernels.py:23 layout). */
int epb_fifo_ctl(epb_t* ctx, int channel, int64_t** host_ctl, int64_t* capacity);
int epb_proxy_start(epb_t* ctx);
int epb_proxy_stop(epb_t* ctx);
/* Proxy counters: commands served, copies issued, atomics issued. */
int epb_proxy_stats(epb_t* ctx, int64_t* out3);
/* Device-side FIFO microbench: `num_cmds` WRITE commands pushed by one producer
 * warp per channel (device push + check_completion), drained by the proxy in
 * "count only" mode.  elapsed_ns receives device time. */
int epb_fifo_device_bench(epb_t* ctx, int64_t num_cmds, int channels, int64_t* elapsed_ns, void* stream);

/* ---- Barrier TransferCmd ---------------
 * The proxies' all-peer barrier: one shared-memory segment per job (ranks of one
 * node), an epoch flag per rank.  Replaces the reference's barrier protocol
 * (epsim models it in its transport simulator only).
 * epb_barrier_*: the host rendezvous itself (also usable without a GPU).
 * epb_proxy_barrier: stream-ordered GPU-side barrier: a kernel pushes a BARRIER
 * command on `channel` and spins on check_completion of its index; the proxy
 * completes it once every rank's proxy has entered (same_rail != 0: SameRail
 * scope, which has no peers on one node and completes at once). */
typedef struct epb_barrier epb_barrier_t;
int epb_barrier_open(const char* name, int world, int rank, epb_barrier_t** out);
int epb_barrier_wait(epb_barrier_t* b, int same_rail, double timeout_s);
int epb_barrier_close(epb_barrier_t* b, int unlink_segment);
int epb_proxy_barrier(epb_t* ctx, int channel, int same_rail, void* stream);

/* Drain(Idx): a kernel pushes a DRAIN command
 * on `channel` (length_or_value = upto + 1; upto < 0: everything issued so far)
 * and spins on check_completion of it; the proxy completes it once every copy
 * issued for commands <= upto of that channel has landed.  Blocking on the GPU
 * side, stream-ordered. */
int epb_proxy_drain(epb_t* ctx, int channel, int64_t upto, void* stream);
/* Test producer for Drain(Idx): a kernel pushes n WRITEs (block i of `bytes`
 * from src_off + i*bytes to dst_off + i*bytes at rank dst, arena offsets) then
 * Drain(upto-th of them); after it completes, result[i] (device int32 [n+1]) =
 * 1 if block i had landed, result[n] = ns from the drain push to completion. */
int epb_debug_drain_test(epb_t* ctx, int channel, int dst, int n, int64_t src_off, int64_t dst_off, int64_t bytes,
                         int64_t upto, int32_t* result, void* stream);

/* Phase trace of a STOPPED proxy (EPB_TRACE=1): rows of 4 int64 {host
 * CLOCK_REALTIME ns, kind, a, b}; kind 1 = tail seen (a = channel, b = tail),
 * 2 = copy issued (a = dst, b = bytes), 3 = value write issued (a = dst,
 * b = value), 4 = COMPLETED published (a = channel, b = value).  Returns the
 * number of events (copies min(n, max_events) into out). */
int64_t epb_proxy_trace(epb_t* ctx, int64_t* out, int64_t max_events);

/* %globaltimer - CLOCK_REALTIME offset (ns) and its uncertainty, for lining up
 * kernel phase marks with the proxy's host events. */
int epb_clock_calibrate(int64_t* offset_ns, int64_t* error_ns);

#ifdef __cplusplus
}
#endif
#endif /* EPB_H_ */
