// stream_microbench.cu — HBM streaming-read rates of the primitives the FFN
// can be built from: 1-D bulk copies (cp.async.bulk) into an smem ring with
// and without consumer work, versus plain 16-byte LDG loops.
#include <cstdio>
#include <cstdint>
#include "ffn_tma.cuh"

using namespace moeb;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int TOUCH>
__global__ void __launch_bounds__(288, 1) bulk_stream(const uint8_t* src, size_t bytes, uint32_t chunk, uint32_t stages, float* out) {
  extern __shared__ __align__(16) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t per = bytes / gridDim.x / chunk * chunk;
  const uint8_t* base = src + per * blockIdx.x;
  const uint32_t n = (uint32_t)(per / chunk);
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t st = 0, ph = 0;
      for (uint32_t i = 0; i < n; ++i) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect_tx(&full[st], chunk);
        bulk_g2s(ring + st * chunk, base + (size_t)i * chunk, chunk, &full[st], pol);
        if (++st == stages) { st = 0; ph ^= 1; }
      }
    }
  } else {
    uint32_t st = 0, ph = 0;
    float acc = 0.f;
    for (uint32_t i = 0; i < n; ++i) {
      mbar_wait(&full[st], ph);
      if (TOUCH) {
        const uint4* p = reinterpret_cast<const uint4*>(ring + st * chunk);
        for (uint32_t j = (warp - 1) * 32 + lane; j < chunk / 16; j += 256) {
          const uint4 v = p[j];
          acc += __uint_as_float(v.x) + __uint_as_float(v.w);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == stages) { st = 0; ph ^= 1; }
    }
    if (acc == 1.2345f) out[0] = acc;
  }
}

__global__ void ldg_stream(const uint4* src, size_t n16, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride * 8) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) if (i + j * stride < n16) v[j] = ldg_cg(src + i + j * stride);
#pragma unroll
    for (int j = 0; j < 8; ++j) if (i + j * stride < n16) acc += __uint_as_float(v[j].x);
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const size_t bytes = 1ull << 30;
  uint8_t* src;
  float* out;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(src, 1, bytes));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto fn) {
    fn();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return bytes * 5 / (ms * 1e-3) / 1e9;
  };
  for (uint32_t chunk : {8192u, 16384u, 32768u}) {
    for (uint32_t stages : {2u, 4u, 6u}) {
      const size_t smem = (size_t)chunk * stages;
      if (smem > 200 * 1024) continue;
      cudaFuncSetAttribute(bulk_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(bulk_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const double g0 = timeit([&] { bulk_stream<0><<<sms, 288, smem>>>(src, bytes, chunk, stages, out); });
      const double g1 = timeit([&] { bulk_stream<1><<<sms, 288, smem>>>(src, bytes, chunk, stages, out); });
      printf("bulk chunk=%5u stages=%u: no-touch %.0f GB/s, touch %.0f GB/s\n", chunk, stages, g0, g1);
    }
  }
  for (int bs : {256, 512, 1024}) {
    for (int per : {1, 2, 4}) {
      const double g = timeit([&] { ldg_stream<<<sms * per, bs>>>((const uint4*)src, bytes / 16, out); });
      printf("ldg grid=%d x %d: %.0f GB/s\n", sms * per, bs, g);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
