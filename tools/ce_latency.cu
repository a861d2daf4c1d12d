// Copy-engine latency probe for the LL proxy transport: how long from the host
// issuing cudaMemcpyAsync (GPU0 -> GPU1 peer) + cuStreamWriteValue64 until the
// signal is visible, as a function of bytes and of how many streams the bytes
// are split over.  The signal goes to pinned host memory, so the figure is an
// upper bound on the device-side landing time (+ ~1 us PCIe write).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/ce_latency.cu -o /tmp/ce_latency
//   ./ce_latency [dst_dev]   (dst_dev 0 = local copy, 1 = peer; default 1)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

using WV64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const int dst_dev = argc > 1 ? std::atoi(argv[1]) : 1;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (dst_dev >= ndev) {
    std::printf("need %d GPUs\n", dst_dev + 1);
    return 0;
  }
  CK(cudaSetDevice(0));
  if (dst_dev != 0) CK(cudaDeviceEnablePeerAccess(dst_dev, 0));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q));
  WV64 wv = reinterpret_cast<WV64>(p);
  const size_t kMax = 16u << 20;
  void* src = nullptr;
  void* dst = nullptr;
  CK(cudaMalloc(&src, kMax));
  CK(cudaSetDevice(dst_dev));
  CK(cudaMalloc(&dst, kMax));
  CK(cudaSetDevice(0));
  const int kMaxStreams = 8;
  volatile uint64_t* flags = nullptr;
  CK(cudaHostAlloc((void**)&flags, 64 * sizeof(uint64_t), cudaHostAllocMapped));
  uint64_t* dflags = nullptr;
  CK(cudaHostGetDevicePointer((void**)&dflags, (void*)flags, 0));
  for (int i = 0; i < 64; ++i) flags[i] = 0;
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  for (int prio = 0; prio < 2; ++prio) {
    std::vector<cudaStream_t> st(kMaxStreams);
    for (auto& s : st) CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio ? hi : lo));
    uint64_t it = 0;
    std::printf("# dst_dev %d priority %s\n# bytes streams issue_us(med) signal_us(med) signal_us(p90) GB/s\n", dst_dev,
                prio ? "high" : "default");
    for (size_t bytes : {size_t(0), size_t(16) << 10, size_t(128) << 10, size_t(512) << 10, size_t(1) << 20,
                         size_t(4) << 20, size_t(16) << 20}) {
      for (int ns : {1, 2, 4, 8}) {
        std::vector<double> iss, sig;
        for (int rep = 0; rep < 60; ++rep) {
          ++it;
          const size_t per = (bytes / ns + 255) & ~size_t(255);
          const double t0 = now_us();
          for (int s = 0; s < ns; ++s) {
            if (per)
              CK(cudaMemcpyAsync((char*)dst + s * per, (char*)src + s * per, std::min(per, kMax - s * per),
                                 cudaMemcpyDeviceToDevice, st[s]));
            if (wv(st[s], (CUdeviceptr)(dflags + s), it, 0) != CUDA_SUCCESS) {
              std::printf("writevalue failed\n");
              return 1;
            }
          }
          const double t1 = now_us();
          for (int s = 0; s < ns; ++s)
            while (flags[s] < it) {
            }
          const double t2 = now_us();
          if (rep >= 10) {
            iss.push_back(t1 - t0);
            sig.push_back(t2 - t0);
          }
        }
        std::sort(iss.begin(), iss.end());
        std::sort(sig.begin(), sig.end());
        const double med = sig[sig.size() / 2];
        std::printf("%9zu %2d %7.2f %8.2f %8.2f %7.1f\n", bytes, ns, iss[iss.size() / 2], med,
                    sig[sig.size() * 9 / 10], bytes / med / 1e3);
      }
    }
    for (auto& s : st) CK(cudaStreamDestroy(s));
  }
  return 0;
}
