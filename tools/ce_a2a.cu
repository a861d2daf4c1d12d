// All-to-all copy-engine probe for the LL proxy transport: every GPU moves
// `bytes` to each of its peers at once (one host thread per GPU, like one
// proxy per rank) and the time until every signal is visible is measured for
// four ways of arranging the copies and the stream-ordered signals:
//   A  one stream per peer: copy, signal            (the shipped proxy)
//   B  one stream: all copies, then all signals
//   C  one stream: copy, signal, copy, signal, ...
//   D  receiver pull: one stream on the receiver copies from every peer, then
//      one local signal
//   K  SM copy kernel: one launch per GPU copies to every peer (blocks split
//      each peer's bytes) and the last block per peer writes its signal
//   L  as K, one launch per peer
// Signals go to pinned host memory (cuStreamWriteValue64), so times include
// ~1 us of PCIe write.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/ce_a2a.cu -o /tmp/ce_a2a -lpthread
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));  \
      std::exit(1);                                                                             \
    }                                                                                           \
  } while (0)

using WV64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
static WV64 wv;

__global__ void kcopy(const int4* const* src, int4* const* dst, unsigned long long* const* flag, uint64_t it,
                      uint64_t n16, int bpp, unsigned* tickets) {
  const int p = blockIdx.x / bpp, b = blockIdx.x % bpp;
  const uint64_t u0 = n16 * b / bpp, u1 = n16 * (b + 1) / bpp;
  for (uint64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
    int4 v;
    asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src[p] + u));
    dst[p][u] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(&tickets[p], 1u) == (unsigned)bpp - 1) {
      tickets[p] = 0;
      __threadfence_system();
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag[p]), "l"(it) : "memory");
    }
  }
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

constexpr int kMaxG = 8;
struct Gpu {
  char* buf = nullptr;  // [kMaxG send slots | kMaxG recv slots] of `slot` bytes
  cudaStream_t st[kMaxG];
};

int main(int argc, char** argv) {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  G = std::min(G, argc > 1 ? std::atoi(argv[1]) : kMaxG);
  if (G < 2) {
    std::printf("need 2 GPUs\n");
    return 0;
  }
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q));
  wv = reinterpret_cast<WV64>(p);
  const size_t slot = 4u << 20;
  std::vector<Gpu> g(G);
  for (int i = 0; i < G; ++i) {
    CK(cudaSetDevice(i));
    for (int j = 0; j < G; ++j)
      if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
    CK(cudaMalloc(&g[i].buf, 2 * kMaxG * slot));
    for (int s = 0; s < kMaxG; ++s) CK(cudaStreamCreateWithFlags(&g[i].st[s], cudaStreamNonBlocking));
  }
  volatile uint64_t* flags = nullptr;
  CK(cudaHostAlloc((void**)&flags, kMaxG * kMaxG * sizeof(uint64_t), cudaHostAllocMapped | cudaHostAllocPortable));
  uint64_t* dflags = nullptr;
  CK(cudaHostGetDevicePointer((void**)&dflags, (void*)flags, 0));
  for (int i = 0; i < kMaxG * kMaxG; ++i) flags[i] = 0;

  std::atomic<int> arrive{0};
  std::atomic<uint64_t> go{0};
  std::printf("# GPUs %d\n# mode bytes_per_peer median_us p90_us (max over GPUs of issue->all own signals seen)\n", G);
  for (size_t bytes : {size_t(64) << 10, size_t(512) << 10, size_t(1) << 20, size_t(2) << 20}) {
    for (char mode : {'A', 'K', 'L'}) {
      const int reps = 60;
      std::vector<std::vector<double>> lat(G);
      uint64_t base_it = 0;
      static uint64_t it_global = 0;
      base_it = it_global;
      it_global += reps;
      auto worker = [&](int i) {
        CK(cudaSetDevice(i));
        for (int r = 0; r < reps; ++r) {
          const uint64_t it = base_it + r + 1;
          // rendezvous: every thread starts the iteration together
          if (arrive.fetch_add(1) + 1 == G * (int)(it - base_it)) go.store(it);
          while (go.load() < it) {
          }
          const double t0 = now_us();
          int nsig = 0;
          auto sig = [&](cudaStream_t s, int slot_id) {
            if (wv((CUstream)s, (CUdeviceptr)(dflags + i * kMaxG + slot_id), it, 0) != CUDA_SUCCESS) std::exit(2);
            ++nsig;
          };
          auto copy_to = [&](int j, cudaStream_t s) {  // push: my send slot j -> j's recv slot i
            CK(cudaMemcpyAsync(g[j].buf + (kMaxG + i) * slot, g[i].buf + j * slot, bytes, cudaMemcpyDefault, s));
          };
          int k = 0;
          if (mode == 'A') {
            for (int j = 0; j < G; ++j)
              if (j != i) {
                copy_to(j, g[i].st[k]);
                sig(g[i].st[k], k);
                ++k;
              }
          } else if (mode == 'B') {
            for (int j = 0; j < G; ++j)
              if (j != i) copy_to(j, g[i].st[0]);
            for (int j = 0; j < G; ++j)
              if (j != i) sig(g[i].st[0], k++);
          } else if (mode == 'C') {
            for (int j = 0; j < G; ++j)
              if (j != i) {
                copy_to(j, g[i].st[0]);
                sig(g[i].st[0], k++);
              }
          } else if (mode == 'K' || mode == 'L') {
            static thread_local const int4** d_src = nullptr;
            static thread_local int4** d_dst = nullptr;
            static thread_local unsigned long long** d_flag = nullptr;
            static thread_local unsigned* d_tick = nullptr;
            if (!d_src) {
              CK(cudaMallocManaged(&d_src, sizeof(void*) * kMaxG));
              CK(cudaMallocManaged(&d_dst, sizeof(void*) * kMaxG));
              CK(cudaMallocManaged(&d_flag, sizeof(void*) * kMaxG));
              CK(cudaMalloc(&d_tick, sizeof(unsigned) * kMaxG * kMaxG));
              CK(cudaMemset(d_tick, 0, sizeof(unsigned) * kMaxG * kMaxG));
              int q = 0;
              for (int j = 0; j < G; ++j)
                if (j != i) {
                  d_src[q] = reinterpret_cast<const int4*>(g[i].buf + j * slot);
                  d_dst[q] = reinterpret_cast<int4*>(g[j].buf + (kMaxG + i) * slot);
                  d_flag[q] = reinterpret_cast<unsigned long long*>(dflags + i * kMaxG + q);
                  ++q;
                }
              CK(cudaDeviceSynchronize());
            }
            const int bpp = std::max<int>(1, (int)(bytes >> 16));
            if (mode == 'K') {
              kcopy<<<bpp * (G - 1), 512, 0, g[i].st[0]>>>(d_src, d_dst, d_flag, it, bytes / 16, bpp, d_tick);
            } else {
              for (int q = 0; q < G - 1; ++q)
                kcopy<<<bpp, 512, 0, g[i].st[q]>>>(d_src + q, d_dst + q, d_flag + q, it, bytes / 16, bpp, d_tick + kMaxG * (q + 1));
            }
            nsig = G - 1;
          } else {  // D: pull every peer's send slot for me into my recv slots
            for (int j = 0; j < G; ++j)
              if (j != i)
                CK(cudaMemcpyAsync(g[i].buf + (kMaxG + j) * slot, g[j].buf + i * slot, bytes, cudaMemcpyDefault,
                                   g[i].st[0]));
            sig(g[i].st[0], 0);
          }
          for (int s = 0; s < nsig; ++s)
            while (flags[i * kMaxG + s] < it) {
            }
          lat[i].push_back(now_us() - t0);
        }
      };
      arrive.store(0);
      std::vector<std::thread> th;
      for (int i = 0; i < G; ++i) th.emplace_back(worker, i);
      for (auto& t : th) t.join();
      std::vector<double> worst;
      for (int r = 10; r < reps; ++r) {
        double m = 0;
        for (int i = 0; i < G; ++i) m = std::max(m, lat[i][r]);
        worst.push_back(m);
      }
      std::sort(worst.begin(), worst.end());
      std::printf("%c %8zu %8.2f %8.2f\n", mode, bytes, worst[worst.size() / 2], worst[worst.size() * 9 / 10]);
      std::fflush(stdout);
    }
  }
  return 0;
}
