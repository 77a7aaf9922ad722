// ffn_microbench.cu — isolate the FFN kernel: synthetic plans with N routed
// items (+ optional shared expert) over random weights, timed with CUDA
// events over many launches (weights > L2 between launches via rotation).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2508_18983_b200/csrc \
//        -o tools/ffn_microbench tools/ffn_microbench.cu
#include <cstdio>
#include <vector>

#include "ffn_tma.cuh"

using namespace moeb;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main(int argc, char** argv) {
  const uint32_t d = 2048, F = 1408, S = 2816, B = 1;
  const int n_sets = 24;  // rotate over weight sets so every launch reads from HBM
  const size_t eelems = 3ull * F * d, selems = 3ull * S * d;
  uint16_t* w;
  CK(cudaMalloc(&w, (size_t)n_sets * (64 * eelems + selems) * 2));
  CK(cudaMemset(w, 0x3c, (size_t)n_sets * (64 * eelems + selems) * 2));
  uint16_t *u, *x, *xo;
  float *y, *h;
  uint32_t *ctr, *cd, *fd;
  Plan* plan;
  CK(cudaMalloc(&u, B * d * 2));
  CK(cudaMalloc(&x, B * d * 2));
  CK(cudaMalloc(&xo, B * d * 2));
  CK(cudaMalloc(&y, B * d * 4));
  CK(cudaMalloc(&h, (size_t)kMaxItems * kMaxB * S * 4));
  CK(cudaMalloc(&ctr, (kMaxItems + 2) * 4));
  CK(cudaMalloc(&cd, 4));
  CK(cudaMalloc(&fd, 4));
  CK(cudaMalloc(&plan, kPlanSmem * n_sets));
  CK(cudaMemset(u, 0, B * d * 2));
  CK(cudaMemset(x, 0, B * d * 2));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t dbg = argc > 2 ? atoi(argv[2]) : 0;
  for (int n_routed : {6, 24}) {
    if (argc > 4 && n_routed != atoi(argv[4])) continue;
    for (int shared : {1}) {
      std::vector<Plan> hp(n_sets);
      uint64_t bytes = 0;
      for (int si = 0; si < n_sets; ++si) {
        Plan& p = hp[si];
        memset(&p, 0, sizeof p);
        uint16_t* base = w + (size_t)si * (64 * eelems + selems);
        int n = 0;
        if (shared) {
          Item& it = p.items[n++];
          it.w = base + 64 * eelems; it.F = S; it.n_tok = 1; it.tok[0] = 0; it.wt[0] = 1.f;
        }
        for (int r = 0; r < n_routed; ++r) {
          Item& it = p.items[n++];
          it.w = base + (size_t)r * eelems; it.F = F; it.n_tok = 1; it.tok[0] = 0; it.wt[0] = 0.1f;
        }
        p.n_items = n; p.n_ready = n; p.seq = 1;
        if (si == 0) for (int i = 0; i < n; ++i) bytes += 3ull * p.items[i].F * d * 2;
      }
      CK(cudaMemcpy(plan, hp.data(), kPlanSmem * n_sets, cudaMemcpyHostToDevice));
      const uint32_t SB = argc > 3 ? atoi(argv[3]) * 1024 : 64 * 1024;
      const size_t ubytes = (size_t)B * d * 4;
      const size_t hb = (size_t)(S + 6 * F) * B * 4;
      size_t budget = 220 * 1024 - ubytes - kPlanSmem - hb;
      uint32_t stages = (uint32_t)std::min<size_t>(kMaxStages, budget / SB);
      if (argc > 1 && atoi(argv[1]) > 0) stages = std::min<uint32_t>(stages, atoi(argv[1]));
      size_t smem = (size_t)stages * SB + ubytes + kPlanSmem + hb;
      CK(cudaFuncSetAttribute(ffn_tma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      const int iters = 48;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) {
          cudaMemsetAsync(ctr, 0, (kMaxItems + 2) * 4);
          FfnTArgs f{};
          f.plan = plan + (i % n_sets); f.u = u; f.x_in = x; f.x_out = xo; f.y_out = y; f.h = h; f.ctr = ctr;
          f.copies_done = cd; f.ffn_done = fd; f.B = B; f.d = d; f.Fmax = S; f.stages = stages; f.stage_bytes = SB;
          f.dbg = dbg;
          f.hbuf_bytes = (uint32_t)hb;
          ffn_tma_kernel<1><<<sms, kFfnTThreads, smem>>>(f);
        }
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 1)
          printf("dbg=%u routed=%2d shared=%d stages=%u: %.1f us/launch, %.1f MB, %.0f GB/s (incl memset)\n", dbg, n_routed, shared,
                 stages, ms * 1e3 / iters, bytes / 1e6, bytes / (ms * 1e-3 / iters) / 1e9);
      }
    }
  }
  return 0;
}
