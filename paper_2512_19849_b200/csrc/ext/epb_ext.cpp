// epb_ext.cpp — the per-call host runtime of the Buffer API, in C++.
//
// A pybind11/ATen client of the C ABI (include/epb.h, libepb200.so): it does
// per call what the Python host layer would otherwise do — validate shapes,
// allocate the handle/output tensors, fill the argument structs, launch, wait
// for the receive counts, and hand out zero-copy views of the leased receive
// slot — at a small fraction of the Python cost (the normal-mode step is
// host-bound at one GPU).  Receive slots are leased from a per-rank pool;
// the storage deleter of the views returns the slot, so a slot is reused
// only after every tensor viewing it is gone.
#include <torch/extension.h>
#include <ATen/cuda/CUDAContext.h>
#include <cuda_runtime.h>

#include <chrono>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "epb.h"

namespace py = pybind11;
using at::Tensor;

namespace {

[[noreturn]] void raise_code(int code, const std::string& msg) {
  py::object raise_for = py::module_::import("paper_2512_19849_b200.errors").attr("raise_for");
  raise_for(code, msg);
  throw std::runtime_error(msg);  // raise_for always raises for code != 0
}

inline void check(int rc) {
  if (rc != 0) raise_code(rc, epb_last_error());
}

inline void* dptr(const Tensor& t) { return t.defined() ? t.data_ptr() : nullptr; }
inline void* dptr(const c10::optional<Tensor>& t) { return (t && t->defined()) ? t->data_ptr() : nullptr; }

struct SlotPool {
  std::mutex m;
  std::vector<int> free_slots;
  int scratch = 0;
  std::pair<int, bool> lease() {
    std::lock_guard<std::mutex> g(m);
    if (free_slots.empty()) return {scratch, true};
    int s = free_slots.front();
    free_slots.erase(free_slots.begin());
    return {s, false};
  }
  void release(int s) {
    std::lock_guard<std::mutex> g(m);
    free_slots.push_back(s);
  }
  int num_free() {
    std::lock_guard<std::mutex> g(m);
    return (int)free_slots.size();
  }
};

struct Profiler {
  bool on = false;
  std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t>> ev;
  void begin(cudaEvent_t* s, cudaStream_t st) {
    if (!on) return;
    cudaEventCreate(s);
    cudaEventRecord(*s, st);
  }
  void end(const char* name, cudaEvent_t s, cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.emplace_back(name, s, e);
  }
  py::list collect() {
    py::list out;
    for (auto& t : ev) {
      float ms = 0.f;
      cudaEventSynchronize(std::get<2>(t));
      cudaEventElapsedTime(&ms, std::get<1>(t), std::get<2>(t));
      out.append(py::make_tuple(std::get<0>(t), ms));
      cudaEventDestroy(std::get<1>(t));
      cudaEventDestroy(std::get<2>(t));
    }
    ev.clear();
    return out;
  }
};
Profiler g_prof;

// Host-side phase timers of dispatch (microseconds, cumulative): prepare,
// launch, wait for the counts, build the outputs.  Read with host_timers().
struct HostTimers {
  double t[4] = {0, 0, 0, 0};
  long n = 0;
};
HostTimers g_ht;
using Clock = std::chrono::steady_clock;
inline double us_since(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double, std::micro>(b - a).count();
}

struct Rank {
  uintptr_t ctx = 0;
  int rank = 0, world = 1, num_slots = 1;
  int64_t base = 0;
  int device = 0;
  std::shared_ptr<SlotPool> pool = std::make_shared<SlotPool>();
  std::vector<std::tuple<int, int, epb_recv_layout_t>> layouts;

  Rank(uintptr_t c, int r, int w, int slots, int64_t b, int dev) : ctx(c), rank(r), world(w), num_slots(slots),
                                                                     base(b), device(dev) {
    for (int s = 0; s + 1 < num_slots; ++s) pool->free_slots.push_back(s);
    pool->scratch = num_slots - 1;
  }
  epb_t* h() const { return reinterpret_cast<epb_t*>(ctx); }
  const epb_recv_layout_t& layout(int hidden, int k) {
    for (auto& t : layouts)
      if (std::get<0>(t) == hidden && std::get<1>(t) == k) return std::get<2>(t);
    epb_recv_layout_t L;
    check(epb_recv_layout(h(), hidden, k, &L));
    layouts.emplace_back(hidden, k, L);
    return std::get<2>(layouts.back());
  }
};
using RankP = std::shared_ptr<Rank>;

// One leased receive slot; returned to its pool when the last view is freed.
struct SlotLease {
  std::shared_ptr<SlotPool> pool;
  int slot;
  SlotLease(std::shared_ptr<SlotPool> p, int s) : pool(std::move(p)), slot(s) {}
  ~SlotLease() { pool->release(slot); }
};

std::vector<epb_t*> handles(const std::vector<RankP>& rs) {
  std::vector<epb_t*> v;
  for (auto& r : rs) v.push_back(r->h());
  return v;
}

// ---------------------------------------------------------------------------
py::tuple layout(const Tensor& topk_idx, int num_experts, int num_ranks) {
  TORCH_CHECK(topk_idx.scalar_type() == at::kLong && topk_idx.dim() == 2, "topk_idx must be int64 [T, k]");
  Tensor ti = topk_idx.contiguous();
  const int T = (int)ti.size(0), k = (int)ti.size(1);
  auto opts = ti.options().dtype(at::kInt);
  Tensor counts = at::empty({num_ranks + num_experts}, opts);
  Tensor per_rank = counts.narrow(0, 0, num_ranks);
  Tensor per_expert = counts.narrow(0, num_ranks, num_experts);
  Tensor in_rank = at::empty({T, num_ranks}, ti.options().dtype(at::kBool));
  cudaStream_t st = at::cuda::getCurrentCUDAStream().stream();
  cudaEvent_t s;
  g_prof.begin(&s, st);
  check(epb_get_dispatch_layout(ti.data_ptr<int64_t>(), T, k, num_experts, num_ranks, per_rank.data_ptr<int32_t>(),
                                per_expert.data_ptr<int32_t>(), (uint8_t*)in_rank.data_ptr(), st));
  g_prof.end("layout", s, st);
  return py::make_tuple(per_rank, per_expert, in_rank);
}

// ---------------------------------------------------------------------------
// normal dispatch for a group of (local) ranks
py::list dispatch(const std::vector<RankP>& ranks, const std::vector<Tensor>& xs,
                  const std::vector<c10::optional<Tensor>>& x_scales, const std::vector<Tensor>& in_ranks,
                  const std::vector<c10::optional<Tensor>>& per_experts,
                  const std::vector<c10::optional<Tensor>>& topk_idxs,
                  const std::vector<c10::optional<Tensor>>& topk_ws, int expert_alignment, int num_channels,
                  double timeout_s, int num_worst_tokens = 0) {
  const auto t0 = Clock::now();
  const int n = (int)ranks.size();
  const int R = ranks[0]->world, C = num_channels;
  std::vector<epb_dispatch_args_t> args(n);
  struct St {
    Tensor x, xs, ir, pe, ti, tw, hbuf;
    int T, H, k, E, elem, slot;
    bool copy_out;
    const epb_recv_layout_t* lay;
  };
  std::vector<St> st(n);
  for (int i = 0; i < n; ++i) {
    St& s = st[i];
    s.x = xs[i].contiguous();
    TORCH_CHECK(s.x.dim() == 2, "x must be [T, H]");
    if (s.x.scalar_type() == at::kFloat8_e4m3fn) {
      TORCH_CHECK(x_scales[i].has_value(), "FP8 dispatch needs scales");
      s.xs = x_scales[i]->contiguous();
      TORCH_CHECK(s.xs.scalar_type() == at::kFloat && s.xs.dim() == 2, "scales must be float32 [T, H/128]");
      s.elem = 1;
    } else {
      TORCH_CHECK(s.x.scalar_type() == at::kBFloat16, "dispatch expects bf16 x or an (fp8, scales) tuple");
      s.elem = 2;
    }
    s.T = (int)s.x.size(0);
    s.H = (int)s.x.size(1);
    s.ir = in_ranks[i].contiguous();
    TORCH_CHECK(s.ir.scalar_type() == at::kBool && s.ir.dim() == 2 && s.ir.size(0) == s.T && s.ir.size(1) == R,
                "is_token_in_rank must be bool [num_tokens, num_ranks]");
    s.k = 0;
    s.E = 0;
    if (topk_idxs[i].has_value() && topk_idxs[i]->defined()) {
      s.ti = topk_idxs[i]->contiguous();
      s.k = (int)s.ti.size(1);
      if (topk_ws[i].has_value() && topk_ws[i]->defined()) s.tw = topk_ws[i]->to(at::kFloat).contiguous();
      TORCH_CHECK(per_experts[i].has_value() && per_experts[i]->defined(),
                  "num_tokens_per_expert is required with topk_idx");
    }
    if (per_experts[i].has_value() && per_experts[i]->defined()) {
      s.pe = per_experts[i]->contiguous();
      s.E = (int)s.pe.numel();
    }
    s.lay = &ranks[i]->layout(s.H, s.k);
    if (num_worst_tokens > s.lay->cap_rows)
      raise_code(EPB_ERR_CONFIG, "num_worst_tokens exceeds the receive slot capacity (num_nvl_bytes)");
    auto lease = ranks[i]->pool->lease();
    s.slot = lease.first;
    s.copy_out = lease.second;
    s.hbuf = at::empty({(int64_t)R * R + 2 * (int64_t)R * C + (int64_t)s.T * R}, s.x.options().dtype(at::kInt));
    int32_t* hb = s.hbuf.data_ptr<int32_t>();
    epb_dispatch_args_t& a = args[i];
    std::memset(&a, 0, sizeof(a));
    a.x = s.x.data_ptr();
    a.x_scales = s.xs.defined() ? s.xs.data_ptr<float>() : nullptr;
    a.hidden = s.H;
    a.elem_bytes = s.elem;
    a.num_scales = s.xs.defined() ? (int)s.xs.size(1) : 0;
    a.topk_idx = s.ti.defined() ? s.ti.data_ptr<int64_t>() : nullptr;
    a.topk_weights = s.tw.defined() ? s.tw.data_ptr<float>() : nullptr;
    a.num_topk = s.k;
    a.is_token_in_rank = (const uint8_t*)s.ir.data_ptr();
    a.num_tokens_per_expert = s.pe.defined() ? s.pe.data_ptr<int32_t>() : nullptr;
    a.num_tokens = s.T;
    a.num_experts = s.E;
    a.expert_alignment = std::max(1, expert_alignment);
    a.recv_slot = s.slot;
    a.rank_prefix_matrix = hb;
    a.channel_prefix_matrix = hb + R * R;
    a.recv_channel_prefix_matrix = hb + R * R + R * C;
    a.send_head = hb + R * R + 2 * R * C;
    a.num_worst_tokens = std::max(0, num_worst_tokens);
  }
  cudaStream_t stream = at::cuda::getCurrentCUDAStream().stream();
  auto hs = handles(ranks);
  std::vector<int64_t> nrecv(n);
  std::vector<std::vector<int32_t>> per_exp(n);
  {
    cudaEvent_t ev;
    g_prof.begin(&ev, stream);
    const auto t1 = Clock::now();
    int rc = epb_dispatch(hs.data(), n, args.data(), C, stream);
    const auto t2 = Clock::now();
    g_prof.end("dispatch", ev, stream);
    g_ht.t[0] += us_since(t0, t1);
    g_ht.t[1] += us_since(t1, t2);
    for (int i = 0; i < n && rc == 0 && num_worst_tokens <= 0; ++i) {
      const auto tw0 = Clock::now();
      struct Acc {
        Clock::time_point a;
        ~Acc() { g_ht.t[2] += us_since(a, Clock::now()); }
      } acc{tw0};
      const int Lx = st[i].E ? st[i].E / R : 0;
      per_exp[i].resize(std::max(1, Lx));
      py::gil_scoped_release nogil;
      rc = epb_wait_notify(hs[i], &nrecv[i], Lx ? per_exp[i].data() : nullptr, Lx, timeout_s);
    }
    if (rc != 0) {
      std::string msg = epb_last_error();
      for (int i = 0; i < n; ++i)
        if (!st[i].copy_out) ranks[i]->pool->release(st[i].slot);
      raise_code(rc, msg);
    }
  }
  const auto t3 = Clock::now();
  py::list out;
  for (int i = 0; i < n; ++i) {
    St& s = st[i];
    Rank& rk = *ranks[i];
    const epb_recv_layout_t& L = *s.lay;
    // num_worst_tokens: no host sync — views of num_worst_tokens rows (rows past
    // the real count carry recv_topk_idx = -1), no per-expert list (DeepEP)
    const int64_t N = num_worst_tokens > 0 ? (int64_t)num_worst_tokens : nrecv[i];
    char* slot_base = reinterpret_cast<char*>(rk.base + L.slot0_off + (int64_t)s.slot * L.slot_bytes);
    const at::Device dev = s.x.device();
    auto opts = s.x.options();
    // zero-copy views of the leased slot: one tensor per output, all sharing
    // the lease; the slot returns to the pool when the last of them is freed
    std::shared_ptr<SlotLease> lease;
    if (!s.copy_out) lease = std::make_shared<SlotLease>(rk.pool, s.slot);
    auto view = [&](int64_t off, at::IntArrayRef sizes, at::ScalarType dt) -> Tensor {
      void* p = slot_base + off;
      if (s.copy_out) return at::for_blob(p, sizes).options(opts.dtype(dt)).target_device(dev).make_tensor().clone();
      return at::for_blob(p, sizes)
          .options(opts.dtype(dt))
          .target_device(dev)
          .deleter([lease](void*) {})
          .make_tensor();
    };
    Tensor recv_x = view(L.off_x, {N, s.H}, s.elem == 2 ? at::kBFloat16 : at::kFloat8_e4m3fn);
    Tensor recv_scales, recv_ti, recv_tw;
    if (s.xs.defined()) recv_scales = view(L.off_scales, {N, s.xs.size(1)}, at::kFloat);
    Tensor recv_src = view(L.off_src_idx, {N}, at::kInt);
    if (s.ti.defined()) {
      recv_ti = view(L.off_topk_idx, {N, s.k}, at::kLong);
      if (s.tw.defined()) recv_tw = view(L.off_topk_w, {N, s.k}, at::kFloat);
    }
    // handle tensors: views of one int32 buffer
    int32_t* hb = s.hbuf.data_ptr<int32_t>();
    Tensor hkeep = s.hbuf;
    auto hview = [&](int64_t off, at::IntArrayRef sizes) -> Tensor {
      return at::for_blob(hb + off, sizes)
          .options(opts.dtype(at::kInt))
          .target_device(dev)
          .deleter([hkeep](void*) {})
          .make_tensor();
    };
    Tensor rpm = hview(0, {R, R});
    Tensor cpm = hview((int64_t)R * R, {R, C});
    Tensor rcpm = hview((int64_t)R * R + R * C, {R, C});
    Tensor send_head = hview((int64_t)R * R + 2 * R * C, {s.T, R});
    py::object px = s.xs.defined() ? py::object(py::make_tuple(recv_x, recv_scales)) : py::cast(recv_x);
    py::object lst = py::none();
    if (s.E && num_worst_tokens > 0) {
      lst = py::list();
    } else if (s.E) {
      const int Lx = s.E / R;
      PyObject* l = PyList_New(Lx);
      if (!l) throw py::error_already_set();
      for (int j = 0; j < Lx; ++j) PyList_SET_ITEM(l, j, PyLong_FromLong(per_exp[i][j]));
      lst = py::reinterpret_steal<py::object>(l);
    }
    py::tuple handle = py::make_tuple(rpm, cpm, rcpm, recv_src, s.ir, send_head);
    out.append(py::make_tuple(px, recv_ti.defined() ? py::cast(recv_ti) : py::none(),
                              recv_tw.defined() ? py::cast(recv_tw) : py::none(), lst, handle));
  }
  const auto t4 = Clock::now();
  g_ht.t[3] += us_since(t3, t4);
  g_ht.n += 1;
  return out;
}

// ---------------------------------------------------------------------------
py::list combine(const std::vector<RankP>& ranks, const std::vector<Tensor>& xs, const std::vector<py::tuple>& hdls,
                 const std::vector<c10::optional<Tensor>>& topk_ws, int num_sms) {
  const int n = (int)ranks.size();
  std::vector<epb_combine_args_t> args(n);
  std::vector<Tensor> keep;
  py::list out;
  for (int i = 0; i < n; ++i) {
    Tensor x = xs[i].contiguous();
    TORCH_CHECK(x.scalar_type() == at::kBFloat16 && x.dim() == 2, "combine expects bf16 x [num_recv_tokens, hidden]");
    Tensor rpm = hdls[i][0].cast<Tensor>(), cpm = hdls[i][1].cast<Tensor>(), rcpm = hdls[i][2].cast<Tensor>(),
           recv_src = hdls[i][3].cast<Tensor>(), ir = hdls[i][4].cast<Tensor>(), sh = hdls[i][5].cast<Tensor>();
    const int N = (int)x.size(0), H = (int)x.size(1), T = (int)ir.size(0);
    if (N != recv_src.numel()) raise_code(EPB_ERR_PROTOCOL, "combine input rows do not match the dispatch handle");
    Tensor w;
    int k = 0;
    if (topk_ws[i].has_value() && topk_ws[i]->defined()) {
      w = topk_ws[i]->to(at::kFloat).contiguous();
      k = (int)w.size(1);
    }
    Tensor o = at::empty({T, H}, x.options());
    Tensor ow = w.defined() ? at::empty({T, k}, w.options()) : Tensor();
    epb_combine_args_t& a = args[i];
    std::memset(&a, 0, sizeof(a));
    a.x = x.data_ptr();
    a.topk_weights = w.defined() ? w.data_ptr<float>() : nullptr;
    a.num_recv = N;
    a.hidden = H;
    a.num_topk = k;
    a.rank_prefix_matrix = rpm.data_ptr<int32_t>();
    a.is_token_in_rank = (const uint8_t*)ir.data_ptr();
    a.send_head = sh.data_ptr<int32_t>();
    a.channel_prefix_matrix = cpm.data_ptr<int32_t>();
    a.recv_channel_prefix_matrix = rcpm.data_ptr<int32_t>();
    a.num_channels = (int)cpm.size(1);
    a.num_tokens = T;
    a.combined_x = o.data_ptr();
    a.combined_topk_weights = ow.defined() ? ow.data_ptr<float>() : nullptr;
    keep.push_back(x);
    keep.push_back(w);
    out.append(py::make_tuple(o, ow.defined() ? py::cast(ow) : py::none()));
  }
  cudaStream_t stream = at::cuda::getCurrentCUDAStream().stream();
  auto hs = handles(ranks);
  cudaEvent_t ev;
  g_prof.begin(&ev, stream);
  check(epb_combine(hs.data(), n, args.data(), num_sms, stream));
  g_prof.end("combine", ev, stream);
  return out;
}

// Single-rank entry points (one process per GPU: the Buffer API), without the
// per-call list packing of the group signatures.
py::tuple dispatch1(const RankP& rank, const Tensor& x, const c10::optional<Tensor>& x_scales, const Tensor& in_rank,
                    const c10::optional<Tensor>& per_expert, const c10::optional<Tensor>& topk_idx,
                    const c10::optional<Tensor>& topk_w, int expert_alignment, int num_channels, double timeout_s,
                    int num_worst_tokens) {
  py::list r = dispatch({rank}, {x}, {x_scales}, {in_rank}, {per_expert}, {topk_idx}, {topk_w}, expert_alignment,
                        num_channels, timeout_s, num_worst_tokens);
  return r[0].cast<py::tuple>();
}

py::tuple combine1(const RankP& rank, const Tensor& x, const py::tuple& handle, const c10::optional<Tensor>& topk_w,
                   int num_sms) {
  py::list r = combine({rank}, {x}, {handle}, {topk_w}, num_sms);
  return r[0].cast<py::tuple>();
}

// ---------------------------------------------------------------------------
// low latency: the call object keeps the argument structs for the recv hook
struct LLCall {
  std::vector<RankP> ranks;
  std::vector<epb_ll_dispatch_args_t> dargs;
  std::vector<epb_ll_combine_args_t> cargs;
  std::vector<Tensor> keep;
  int num_sms = 0;
  bool is_combine = false;
  void recv() {
    auto hs = handles(ranks);
    cudaStream_t stream = at::cuda::getCurrentCUDAStream().stream();
    if (is_combine) {
      for (auto& a : cargs) a.phases = 2;
      check(epb_ll_combine(hs.data(), (int)hs.size(), cargs.data(), num_sms, stream));
    } else {
      for (auto& a : dargs) a.phases = 2;
      check(epb_ll_dispatch(hs.data(), (int)hs.size(), dargs.data(), num_sms, stream));
    }
  }
};

py::tuple ll_dispatch(const std::vector<RankP>& ranks, const std::vector<Tensor>& xs,
                      const std::vector<Tensor>& topk_idxs, int Tm, int E, bool use_fp8, bool round_scale,
                      bool hook, bool use_proxy, int num_sms) {
  const int n = (int)ranks.size();
  const int R = ranks[0]->world;
  TORCH_CHECK(E % R == 0, "num_experts must be a multiple of the number of ranks");
  const int Lx = E / R;
  auto call = std::make_shared<LLCall>();
  call->ranks = ranks;
  call->dargs.resize(n);
  call->num_sms = num_sms;
  py::list res;
  for (int i = 0; i < n; ++i) {
    Tensor x = xs[i].contiguous(), ti = topk_idxs[i].contiguous();
    TORCH_CHECK(x.scalar_type() == at::kBFloat16 && x.dim() == 2, "low_latency_dispatch expects bf16 x [T, H]");
    TORCH_CHECK(ti.scalar_type() == at::kLong && ti.dim() == 2 && ti.size(0) == x.size(0), "topk_idx must be int64 [T, k]");
    const int T = (int)x.size(0), H = (int)x.size(1), k = (int)ti.size(1), S = H / 128;
    if (T > Tm) raise_code(EPB_ERR_CONFIG, "num_tokens exceeds num_max_dispatch_tokens_per_rank");
    auto o = x.options();
    Tensor px = at::empty({Lx, (int64_t)R * Tm, H}, o.dtype(use_fp8 ? at::kFloat8_e4m3fn : at::kBFloat16));
    Tensor ps = use_fp8 ? at::empty({Lx, S, (int64_t)R * Tm}, o.dtype(at::kFloat)) : Tensor();
    Tensor ints = at::empty({Lx + 2 * (int64_t)Lx * R * Tm + (int64_t)T * k}, o.dtype(at::kInt));
    Tensor count = ints.narrow(0, 0, Lx);
    Tensor src_info = ints.narrow(0, Lx, (int64_t)Lx * R * Tm).view({Lx, (int64_t)R * Tm});
    Tensor route = ints.narrow(0, Lx + (int64_t)Lx * R * Tm, (int64_t)Lx * R * Tm).view({Lx, (int64_t)R * Tm});
    Tensor comb_slot = ints.narrow(0, Lx + 2 * (int64_t)Lx * R * Tm, (int64_t)T * k).view({T, k});
    Tensor layout_range = at::empty({Lx, R}, o.dtype(at::kLong));
    epb_ll_dispatch_args_t& a = call->dargs[i];
    std::memset(&a, 0, sizeof(a));
    a.x = x.data_ptr();
    a.topk_idx = ti.data_ptr<int64_t>();
    a.num_tokens = T;
    a.num_topk = k;
    a.hidden = H;
    a.num_experts = E;
    a.max_tokens = Tm;
    a.use_fp8 = use_fp8;
    a.round_scale = round_scale;
    a.packed_recv_x = px.data_ptr();
    a.packed_recv_x_scales = ps.defined() ? ps.data_ptr<float>() : nullptr;
    a.packed_recv_count = count.data_ptr<int32_t>();
    a.packed_recv_src_info = src_info.data_ptr<int32_t>();
    a.packed_recv_layout_range = layout_range.data_ptr<int64_t>();
    a.recv_route = route.data_ptr<int32_t>();
    a.comb_slot = comb_slot.data_ptr<int32_t>();
    a.phases = hook ? 1 : 3;
    a.use_proxy = use_proxy;
    call->keep.insert(call->keep.end(), {x, ti});
    py::object recv = use_fp8 ? py::object(py::make_tuple(px, ps.transpose(1, 2))) : py::cast(px);
    py::tuple handle = py::make_tuple(src_info, layout_range, Tm, H, E, route, comb_slot, count, k, use_proxy);
    res.append(py::make_tuple(recv, count, handle));
  }
  cudaStream_t stream = at::cuda::getCurrentCUDAStream().stream();
  auto hs = handles(ranks);
  cudaEvent_t ev;
  g_prof.begin(&ev, stream);
  check(epb_ll_dispatch(hs.data(), n, call->dargs.data(), num_sms, stream));
  g_prof.end("ll_dispatch", ev, stream);
  return py::make_tuple(res, hook ? py::cast(call) : py::none());
}

py::tuple ll_combine(const std::vector<RankP>& ranks, const std::vector<Tensor>& xs,
                     const std::vector<Tensor>& topk_idxs, const std::vector<Tensor>& topk_ws,
                     const std::vector<py::tuple>& hdls, bool hook, const std::vector<c10::optional<Tensor>>& outs,
                     int num_sms) {
  const int n = (int)ranks.size();
  auto call = std::make_shared<LLCall>();
  call->ranks = ranks;
  call->cargs.resize(n);
  call->num_sms = num_sms;
  call->is_combine = true;
  py::list res;
  for (int i = 0; i < n; ++i) {
    const py::tuple& h = hdls[i];
    Tensor layout_range = h[1].cast<Tensor>(), route = h[5].cast<Tensor>(), comb_slot = h[6].cast<Tensor>(),
           count = h[7].cast<Tensor>();
    const int Tm = h[2].cast<int>(), H = h[3].cast<int>(), E = h[4].cast<int>(), k = h[8].cast<int>();
    const bool use_proxy = h[9].cast<bool>();
    Tensor x = xs[i].contiguous(), ti = topk_idxs[i].contiguous(), w = topk_ws[i].to(at::kFloat).contiguous();
    TORCH_CHECK(x.scalar_type() == at::kBFloat16 && x.dim() == 3 && x.size(2) == H,
                "low_latency_combine expects bf16 x [num_local_experts, R*Tmax, hidden]");
    const int T = (int)comb_slot.size(0);
    if (ti.size(0) != T || ti.size(1) != k || w.size(0) != T || w.size(1) != k)
      raise_code(EPB_ERR_PROTOCOL, "topk_idx / topk_weights do not match the dispatch handle");
    Tensor o = (i < (int)outs.size() && outs[i].has_value() && outs[i]->defined()) ? *outs[i]
                                                                                  : at::empty({T, H}, x.options());
    epb_ll_combine_args_t& a = call->cargs[i];
    std::memset(&a, 0, sizeof(a));
    a.x = x.data_ptr();
    a.topk_idx = ti.data_ptr<int64_t>();
    a.topk_weights = w.data_ptr<float>();
    a.packed_recv_count = count.data_ptr<int32_t>();
    a.packed_recv_layout_range = layout_range.data_ptr<int64_t>();
    a.recv_route = route.data_ptr<int32_t>();
    a.comb_slot = comb_slot.data_ptr<int32_t>();
    a.num_tokens = T;
    a.num_topk = k;
    a.hidden = H;
    a.num_experts = E;
    a.max_tokens = Tm;
    a.combined_x = o.data_ptr();
    a.phases = hook ? 1 : 3;
    a.use_proxy = use_proxy;
    call->keep.insert(call->keep.end(), {x, ti, w});
    res.append(o);
  }
  cudaStream_t stream = at::cuda::getCurrentCUDAStream().stream();
  auto hs = handles(ranks);
  cudaEvent_t ev;
  g_prof.begin(&ev, stream);
  check(epb_ll_combine(hs.data(), n, call->cargs.data(), num_sms, stream));
  g_prof.end("ll_combine", ev, stream);
  return py::make_tuple(res, hook ? py::cast(call) : py::none());
}

}  // namespace

PYBIND11_MODULE(_epb_ext, m) {
  m.doc() = "C++ per-call host runtime of the B200 EP Buffer (client of libepb200.so)";
  py::class_<Rank, RankP>(m, "Rank")
      .def(py::init<uintptr_t, int, int, int, int64_t, int>())
      .def_readonly("ctx", &Rank::ctx)
      .def_readonly("rank", &Rank::rank)
      .def_readonly("world", &Rank::world)
      .def("num_free_slots", [](Rank& r) { return r.pool->num_free(); });
  py::class_<LLCall, std::shared_ptr<LLCall>>(m, "LLCall").def("__call__", &LLCall::recv);
  m.def("layout", &layout);
  m.def("dispatch", &dispatch);
  m.def("combine", &combine);
  m.def("dispatch1", &dispatch1);
  m.def("combine1", &combine1);
  m.def("ll_dispatch", &ll_dispatch);
  m.def("ll_combine", &ll_combine);
  m.def("set_profiling", [](bool on) { g_prof.on = on; });
  m.def("host_timers", []() {
    py::dict d;
    const double n = g_ht.n ? (double)g_ht.n : 1.0;
    d["calls"] = g_ht.n;
    d["prepare_us"] = g_ht.t[0] / n;
    d["launch_us"] = g_ht.t[1] / n;
    d["wait_us"] = g_ht.t[2] / n;
    d["outputs_us"] = g_ht.t[3] / n;
    g_ht = HostTimers();
    return d;
  });
  m.def("collect_profile", []() { return g_prof.collect(); });
}
