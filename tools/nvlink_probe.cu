// nvlink_probe.cu — achievable NVLink write/read bandwidth from SMs on this box.
// Single process, two GPUs with peer access; device 0 kernels move `bytes`
// between local HBM and device 1.  Variants:
//   st   : 16-B vector stores, U loads in flight per lane, G blocks x W warps
//   ld   : 16-B peer loads (pull), local stores
//   tma  : cp.async.bulk global->shared (local) then shared->global (peer), 1 thread per warp
//   ce   : cudaMemcpyPeerAsync
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe tools/nvlink_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>
#include <chrono>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U>
__global__ void st_kernel(const int4* __restrict__ src, int4* dst, size_t n16) {
  const size_t lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
  const size_t chunk = 32 * U;
  for (size_t base = gw * chunk; base < n16; base += nw * chunk) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = base + u * 32 + lane;
      if (i < n16) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = base + u * 32 + lane;
      if (i < n16) asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" :: "l"(dst + i), "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w) : "memory");
    }
  }
}

// TMA 1D bulk: each warp's lane 0 moves CH bytes per step through a 2-stage smem ring
template <int CH>
__global__ void tma_kernel(const char* src, char* dst, size_t bytes) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bar[32][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwb = blockDim.x >> 5;
  char* buf = smem + (size_t)warp * 2 * CH;
  const size_t gw = (size_t)blockIdx.x * nwb + warp, nw = (size_t)gridDim.x * nwb;
  if (lane == 0) {
    for (int s = 0; s < 2; ++s) {
      unsigned a = (unsigned)__cvta_generic_to_shared(&bar[warp][s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (lane != 0) return;
  unsigned phase[2] = {0, 0};
  int it = 0;
  for (size_t off = gw * CH; off < bytes; off += nw * CH, ++it) {
    const int s = it & 1;
    char* b = buf + s * CH;
    unsigned sb = (unsigned)__cvta_generic_to_shared(b);
    unsigned ab = (unsigned)__cvta_generic_to_shared(&bar[warp][s]);
    // make sure the previous bulk store out of this stage has read the smem
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(ab), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(sb), "l"(src + off), "r"(CH), "r"(ab) : "memory");
    // wait load
    unsigned done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(ab), "r"(phase[s]) : "memory");
    }
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + off), "r"(sb), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  size_t bytes = (size_t)(argc > 1 ? atof(argv[1]) : 256) << 20;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  printf("peer access 0->1: %d, bytes %zu MB\n", can, bytes >> 20);
  CK(cudaSetDevice(1));
  char* d1;
  CK(cudaMalloc(&d1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  char *d0, *d0b;
  CK(cudaMalloc(&d0, bytes));
  CK(cudaMalloc(&d0b, bytes));
  CK(cudaMemset(d0, 1, bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto time = [&](auto fn, const char* name) {
    fn();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    const int reps = 10;
    for (int r = 0; r < reps; ++r) fn();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("%-40s %8.1f GB/s\n", name, bytes * reps / (ms / 1e3) / 1e9);
  };
  const size_t n16 = bytes / 16;
  int sms = 148;
  for (int blocksPerSM : {1, 2, 4}) {
    for (int threads : {256, 512, 1024}) {
      if (threads * blocksPerSM > 2048) continue;
      char name[64];
      snprintf(name, sizeof name, "st U=8 %dx%d", sms * blocksPerSM, threads);
      time([&] { st_kernel<8><<<sms * blocksPerSM, threads>>>((int4*)d0, (int4*)d1, n16); }, name);
    }
  }
  time([&] { st_kernel<4><<<sms * 2, 512>>>((int4*)d0, (int4*)d1, n16); }, "st U=4 296x512");
  time([&] { st_kernel<16><<<sms, 512>>>((int4*)d0, (int4*)d1, n16); }, "st U=16 148x512");
  time([&] { st_kernel<8><<<sms, 512>>>((int4*)d0, (int4*)d0b, n16); }, "local copy U=8 148x512");
  time([&] { st_kernel<8><<<sms * 2, 512>>>((int4*)d1, (int4*)d0b, n16); }, "ld (pull) U=8 296x512");
  time([&] { st_kernel<16><<<sms * 2, 512>>>((int4*)d1, (int4*)d0b, n16); }, "ld (pull) U=16 296x512");
  for (int ch : {4096, 8192, 16384}) {
    for (int warps : {4, 8, 16}) {
      size_t smem = (size_t)warps * 2 * ch;
      if (smem > 200 * 1024) continue;
      char name[64];
      snprintf(name, sizeof name, "tma chunk %d, %d warps/blk, %d blk", ch, warps, sms);
      auto k = ch == 4096 ? tma_kernel<4096> : ch == 8192 ? tma_kernel<8192> : tma_kernel<16384>;
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      time([&] { k<<<sms, warps * 32, smem>>>(d0, d1, bytes); }, name);
    }
  }
  time([&] { CK(cudaMemcpyPeerAsync(d1, 1, d0, 0, bytes)); }, "ce cudaMemcpyPeerAsync");

  // bidirectional: both GPUs move `bytes` to / from each other at once
  // (what dispatch / combine do at EP=2); GB/s per direction
  char *s1, *d1b;
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&s1, bytes));
  CK(cudaMalloc(&d1b, bytes));
  CK(cudaMemset(s1, 2, bytes));
  CK(cudaSetDevice(0));
  auto bidir = [&](auto fn0, auto fn1, const char* name) {
    for (int w = 0; w < 2; ++w) {
      CK(cudaSetDevice(0)); fn0();
      CK(cudaSetDevice(1)); fn1();
    }
    CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    const int reps = 10;
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) {
      CK(cudaSetDevice(0)); fn0();
      CK(cudaSetDevice(1)); fn1();
    }
    CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("%-40s %8.1f GB/s per direction\n", name, bytes * reps / s / 1e9);
  };
  bidir([&] { st_kernel<8><<<sms, 512>>>((int4*)d0, (int4*)d1b, n16); },
        [&] { st_kernel<8><<<sms, 512>>>((int4*)s1, (int4*)d0b, n16); }, "bidir st U=8 148x512");
  bidir([&] { st_kernel<8><<<sms * 2, 512>>>((int4*)s1, (int4*)d0b, n16); },
        [&] { st_kernel<8><<<sms * 2, 512>>>((int4*)d0, (int4*)d1b, n16); }, "bidir ld U=8 296x512");
  bidir([&] { st_kernel<16><<<sms * 2, 512>>>((int4*)s1, (int4*)d0b, n16); },
        [&] { st_kernel<16><<<sms * 2, 512>>>((int4*)d0, (int4*)d1b, n16); }, "bidir ld U=16 296x512");
  for (int ch : {4096, 8192, 16384}) {
    auto k = ch == 4096 ? tma_kernel<4096> : ch == 8192 ? tma_kernel<8192> : tma_kernel<16384>;
    for (int warps : {4, 8}) {
      const size_t smem = (size_t)warps * 2 * ch;
      if (smem > 200 * 1024) continue;
      CK(cudaSetDevice(1));
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaSetDevice(0));
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      char name[64];
      snprintf(name, sizeof name, "tma pull chunk %d, %d warps/blk", ch, warps);
      time([&] { k<<<sms, warps * 32, smem>>>(s1, d0b, bytes); }, name);
      snprintf(name, sizeof name, "bidir tma pull chunk %d, %d warps/blk", ch, warps);
      bidir([&] { k<<<sms, warps * 32, smem>>>(s1, d0b, bytes); },
            [&] { k<<<sms, warps * 32, smem>>>(d0, d1b, bytes); }, name);
      snprintf(name, sizeof name, "bidir tma push chunk %d, %d warps/blk", ch, warps);
      bidir([&] { k<<<sms, warps * 32, smem>>>(d0, d1b, bytes); },
            [&] { k<<<sms, warps * 32, smem>>>(s1, d0b, bytes); }, name);
    }
  }
  bidir([&] { CK(cudaMemcpyPeerAsync(d1b, 1, d0, 0, bytes)); },
        [&] { CK(cudaMemcpyPeerAsync(d0b, 0, s1, 1, bytes)); }, "bidir ce");
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
