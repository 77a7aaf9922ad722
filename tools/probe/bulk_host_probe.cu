// One-off probe: cp.async.bulk (the 1-D bulk-copy engine the FFN producers
// use) reading mapped pinned HOST memory into shared memory, vs the copy
// engine. Decides whether an FFN could stream uploads straight over PCIe.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each CTA streams its contiguous share of src through a ring of `stages` x chunk bytes
__global__ void bulk_stream(const unsigned char* src, size_t bytes, uint32_t chunk, uint32_t stages, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t bar[16];
  const size_t per = (bytes / gridDim.x) & ~(size_t)(chunk - 1);
  const unsigned char* base = src + blockIdx.x * per;
  const uint32_t n = (uint32_t)(per / chunk);
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    unsigned long long acc = 0;
    for (uint32_t i = 0; i < n + stages; ++i) {
      if (i >= stages) {  // consume chunk i - stages
        const uint32_t s = (i - stages) % stages, ph = ((i - stages) / stages) & 1;
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(sa(&bar[s])), "r"(ph) : "memory");
        acc += ring[s * chunk];
      }
      if (i < n) {
        const uint32_t s = i % stages;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(ring + s * chunk)), "l"(base + (size_t)i * chunk), "r"(chunk), "r"(sa(&bar[s])) : "memory");
      }
    }
    sink[blockIdx.x] = acc;
  }
}

int main() {
  const size_t bytes = 256ull << 20;
  unsigned char* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  for (size_t i = 0; i < bytes; i += 4096) h[i] = (unsigned char)i;
  unsigned char* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  unsigned char* d;
  CK(cudaMalloc(&d, bytes));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 4096 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  cudaEventRecord(e0);
  for (int r = 0; r < 4; ++r) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("CE H2D 256MB x4: %.2f GB/s\n", 4 * bytes / (ms * 1e-3) / 1e9);
  const uint32_t chunks[] = {4096, 12288, 16384, 32768};
  const uint32_t grids[] = {16, 74, 148};
  for (uint32_t chunk : chunks)
    for (uint32_t g : grids) {
      const uint32_t stages = chunk >= 32768 ? 6 : 12;
      const size_t smem = (size_t)stages * chunk;
      CK(cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      bulk_stream<<<g, 32, smem>>>(hd, bytes, chunk, stages, sink);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 4; ++r) bulk_stream<<<g, 32, smem>>>(hd, bytes, chunk, stages, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      cudaEventElapsedTime(&ms, e0, e1);
      const size_t moved = 4ull * g * ((bytes / g) & ~(size_t)(chunk - 1));
      printf("bulk host->smem chunk %u B, %u stages, grid %u: %.2f GB/s\n", chunk, stages, g, moved / (ms * 1e-3) / 1e9);
    }
  return 0;
}
