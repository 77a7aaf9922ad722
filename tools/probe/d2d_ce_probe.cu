// One-off probe: does a device-to-device cudaMemcpyAsync make progress while a
// persistent kernel occupies every SM (i.e. does it run on a copy engine or as
// an SM kernel)? Variants: a device-to-device copy, and the same bytes staged
// through pinned host memory (two copy-engine hops). The spinning kernel gives
// up after 2 s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void spin(volatile uint32_t* flag, uint32_t want, uint32_t* result) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag != want) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) { if (threadIdx.x == 0) atomicExch(result, 1u); return; }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(result, 2u);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = 17301504;
  void *a, *b;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  uint32_t *flag, *res;
  CK(cudaMalloc(&flag, 4));
  CK(cudaMallocHost(&res, 4));
  void* hbuf;
  CK(cudaMallocHost(&hbuf, bytes));
  cudaStream_t sk, sc;
  CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  const size_t sizes[3] = {196608, 1u << 20, bytes};
  for (int vs = 0; vs < 6; ++vs) {
    const int variant = vs & 1;
    const size_t nb = sizes[vs >> 1];
    CK(cudaMemset(flag, 0, 4));
    *res = 0;
    CK(cudaDeviceSynchronize());
    // one CTA per SM with all of the opt-in shared memory (as the FFN grids
    // use ~224 KB): nothing else fits on any SM
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
    CK(cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    spin<<<sms, 1024, optin, sk>>>(flag, 7u, res);
    CK(cudaGetLastError());
    if (variant == 0) {
      CK(cudaMemcpyAsync(b, a, nb, cudaMemcpyDeviceToDevice, sc));
    } else {
      CK(cudaMemcpyAsync(hbuf, a, nb, cudaMemcpyDeviceToHost, sc));
      CK(cudaMemcpyAsync(b, hbuf, nb, cudaMemcpyHostToDevice, sc));
    }
    CUdeviceptr fp = (CUdeviceptr)flag;
    if (cuStreamWriteValue32(sc, fp, 7u, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) printf("writevalue failed\n");
    CK(cudaDeviceSynchronize());
    printf("%zu B, %s: %s\n", nb, variant == 0 ? "cudaMemcpyAsync D2D" : "D2H + H2D through pinned memory",
           *res == 2 ? "progressed beside the persistent kernel (copy engine)" : "blocked until the kernel gave up (SM copy)");
  }
  return 0;
}
