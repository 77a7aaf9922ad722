// One-off probe: HBM read throughput of cp.async.bulk streams (one producer
// lane per CTA, mbarrier ring, a consumer warp that only waits and releases)
// vs bulk-copy size and ring depth: do the decode FFN's 12 KB row copies cap
// the stream below larger copies?
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
}

__global__ void stream(const unsigned char* src, size_t per_cta, uint32_t chunk, uint32_t stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  const unsigned char* base = src + blockIdx.x * per_cta;
  const uint32_t n = (uint32_t)(per_cta / chunk);
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // producer
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % stages;
      if (i >= stages) wait_bar(&empty[s], ((i / stages) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                   ::"r"(sa(ring + (size_t)s * chunk)), "l"(base + (size_t)i * chunk), "r"(chunk), "r"(sa(&full[s])), "l"(pol)
                   : "memory");
    }
  } else if (threadIdx.x == 32) {  // consumer
    unsigned long long acc = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % stages;
      wait_bar(&full[s], (i / stages) & 1);
      acc += ring[(size_t)s * chunk + (i & 127)];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
    sink[blockIdx.x] = acc;
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t total = 4ull << 30;  // 4 GB: rotate through it, never L2-resident
  unsigned char* buf;
  CK(cudaMalloc(&buf, total));
  CK(cudaMemset(buf, 1, total));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 4096 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t chunks[] = {12288, 24576, 36864, 49152};
  const uint32_t depth_bytes[] = {96 << 10, 192 << 10};
  const size_t per_launch = 141ull << 20;  // ~ one decode FFN launch
  for (uint32_t ch : chunks)
    for (uint32_t db : depth_bytes) {
      const uint32_t stages = db / ch < 32 ? db / ch : 32;
      if (stages < 2) continue;
      const size_t smem = (size_t)stages * ch;
      CK(cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const size_t per_cta = (per_launch / sms) / ch * ch;
      const int reps = 20;
      float best = 1e9f;
      for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) {
          const size_t off = ((size_t)r * per_cta * sms) % (total - per_cta * sms);
          stream<<<sms, 64, smem>>>(buf + off, per_cta, ch, stages, sink);
        }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double bytes = (double)per_cta * sms * reps;
      printf("chunk %6u B x %2u stages (%3u KB in flight/SM): %7.1f GB/s, %.2f us per 141 MB launch\n", ch, stages,
             stages * ch / 1024, bytes / (best * 1e-3) / 1e9, best * 1e3 / reps);
    }
  return 0;
}
