// One-off hardware probe: pinned H2D copy-engine bandwidth vs SM-driven
// zero-copy reads of mapped host memory, and HBM copy bandwidth. Used to pick
// the expert-upload engine.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U>
__global__ void __launch_bounds__(1024) zc_copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = tid; base < n16; base += stride * U) {
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      size_t i = base + j * stride;
      if (i < n16) v[j] = __ldcs(src + i);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      size_t i = base + j * stride;
      if (i < n16) dst[i] = v[j];
    }
  }
}

// contiguous per-CTA chunking (better for PCIe read combining?)
template <int U>
__global__ void __launch_bounds__(1024) zc_copy_chunk(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t per = (n16 + gridDim.x - 1) / gridDim.x;
  size_t lo = blockIdx.x * per, hi = min(n16, lo + per);
  for (size_t base = lo + threadIdx.x; base < hi; base += (size_t)blockDim.x * U) {
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      size_t i = base + j * blockDim.x;
      if (i < hi) v[j] = __ldcs(src + i);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      size_t i = base + j * blockDim.x;
      if (i < hi) dst[i] = v[j];
    }
  }
}

int main() {
  const size_t bytes = 256ull << 20;
  void *h, *d, *d2;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 1, bytes);
  CK(cudaMalloc(&d, bytes));
  CK(cudaMalloc(&d2, bytes));
  void* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  // best-of-reps duration (ms); NaN when a launch or the stream failed, so
  // a failed configuration can never print as a bandwidth
  auto timeit = [&](auto fn, int reps) {
    float best = 1e9;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(a, s); fn();
      if (cudaGetLastError() != cudaSuccess) return NAN;
      cudaEventRecord(b, s);
      if (cudaEventSynchronize(b) != cudaSuccess) return NAN;
      float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
    }
    return best;
  };
  float ms = timeit([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s); }, 10);
  printf("CE H2D 256MB: %.2f GB/s\n", bytes / ms / 1e6);
  ms = timeit([&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s); }, 10);
  printf("CE D2H 256MB: %.2f GB/s\n", bytes / ms / 1e6);
  const size_t eb = 17301504;
  ms = timeit([&] { for (int i = 0; i < 14; ++i) cudaMemcpyAsync((char*)d + i * eb, (char*)h + i * eb, eb, cudaMemcpyHostToDevice, s); }, 10);
  printf("CE H2D 14x17.3MB: %.2f GB/s\n", 14 * eb / ms / 1e6);
  ms = timeit([&] { cudaMemcpyAsync(d, h, eb, cudaMemcpyHostToDevice, s); }, 20);
  printf("CE H2D 1x17.3MB: %.2f GB/s (%.1f us)\n", eb / ms / 1e6, ms * 1e3);
  ms = timeit([&] { cudaMemcpyAsync(d2, d, bytes, cudaMemcpyDeviceToDevice, s); }, 10);
  printf("D2D 256MB: %.2f GB/s (r+w)\n", 2 * bytes / ms / 1e6);
  size_t n16 = bytes / 16;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g : {sms, 2 * sms, 4 * sms, 8 * sms, 16 * sms}) {
    for (int bs : {256, 512, 1024}) {
      ms = timeit([&] { zc_copy<8><<<g, bs, 0, s>>>((const int4*)hd, (int4*)d, n16); }, 5);
      float ms2 = timeit([&] { zc_copy_chunk<8><<<g, bs, 0, s>>>((const int4*)hd, (int4*)d, n16); }, 5);
      float ms3 = timeit([&] { zc_copy<16><<<g, bs, 0, s>>>((const int4*)hd, (int4*)d, n16); }, 5);
      printf("ZC grid=%d bs=%d: strided U8 %.2f GB/s, chunk U8 %.2f GB/s, strided U16 %.2f GB/s\n", g, bs,
             bytes / ms / 1e6, bytes / ms2 / 1e6, bytes / ms3 / 1e6);
    }
  }
  // small grids: how much PCIe BW can few SMs pull
  for (int g : {8, 16, 32, 64}) {
    ms = timeit([&] { zc_copy_chunk<16><<<g, 1024, 0, s>>>((const int4*)hd, (int4*)d, n16); }, 5);
    printf("ZC few-SM grid=%d bs=1024 chunk U16: %.2f GB/s\n", g, bytes / ms / 1e6);
  }
  // concurrent CE + ZC on two streams
  cudaStream_t s2; cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t j; cudaEventCreate(&j);
  ms = timeit([&] {
    cudaEventRecord(j, s); cudaStreamWaitEvent(s2, j, 0);
    cudaMemcpyAsync(d2, h, bytes / 2, cudaMemcpyHostToDevice, s2);
    zc_copy_chunk<8><<<2 * sms, 512, 0, s>>>((const int4*)((char*)hd + bytes / 2), (int4*)d, n16 / 2);
    cudaEventRecord(j, s2); cudaStreamWaitEvent(s, j, 0);
  }, 5);
  printf("CE+ZC concurrent 256MB total: %.2f GB/s\n", bytes / ms / 1e6);
  // HBM read-only GEMV-like streaming check
  ms = timeit([&] { zc_copy<8><<<4 * sms, 512, 0, s>>>((const int4*)d, (int4*)d2, n16); }, 10);
  printf("SM copy HBM->HBM 256MB: %.2f GB/s (r+w)\n", 2 * bytes / ms / 1e6);
  return 0;
}
