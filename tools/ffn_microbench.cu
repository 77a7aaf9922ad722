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
  CK(cudaMalloc(&ctr, kFfnCtrWords * 4));
  CK(cudaMalloc(&cd, 4));
  CK(cudaMalloc(&fd, 4));
  CK(cudaMalloc(&plan, kPlanSmem * n_sets));
  uint64_t* tsd;
  CK(cudaMalloc(&tsd, 8 * 8 * 1024));
  CK(cudaMemset(tsd, 0, 8 * 8 * 1024));
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
      FfnLaunch fl = ffn_launch_config(B, d, F, S, 64, n_routed, sms);
      if (argc > 1 && atoi(argv[1]) > 0) fl.stages = std::min<uint32_t>(fl.stages, atoi(argv[1]));
      const size_t smem = fl.smem - 0;
      CK(cudaFuncSetAttribute(fl.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      const int iters = 48;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) {
          cudaMemsetAsync(ctr, 0, kFfnCtrWords * 4);
          FfnTArgs f{};
          f.plan = plan + (i % n_sets); f.u = u; f.x_in = x; f.x_out = xo; f.y_out = y; f.h = h; f.ctr = ctr;
          f.copies_done = cd; f.ffn_done = fd; f.B = B; f.d = d; f.Fmax = S; f.stages = fl.stages;
          f.stage_bytes = fl.stage_bytes; f.acc_rows = fl.acc_rows; f.plan_smem = fl.plan_smem; f.x_smem = fl.x_smem; f.dbg = dbg; f.hbuf_bytes = fl.hbuf_bytes;
          f.tstamp = (rep == 1 && i == iters - 1) ? tsd : nullptr;
          fl.fn<<<sms, fl.threads, smem>>>(f);
        }
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 1) {
        std::vector<uint64_t> t(8 * sms);
        CK(cudaMemcpy(t.data(), tsd, 8 * 8 * sms, cudaMemcpyDeviceToHost));
        uint64_t t0 = ~0ull;
        for (int i = 0; i < sms; ++i) t0 = std::min(t0, t[i * 8]);
        const char* nm[8] = {"start", "prologue", "first_stage", "gu_done", "barrier", "consumers_done", "end", "pre_atomic"};
        for (int k = 0; k < 8; ++k) {
          double mn = 1e30, mx = 0, avg = 0;
          for (int i = 0; i < sms; ++i) { double v = (t[i * 8 + k] - t0) * 1e-3; mn = std::min(mn, v); mx = std::max(mx, v); avg += v / sms; }
          printf("   %-15s min %7.2f avg %7.2f max %7.2f us\n", nm[k], mn, avg, mx);
        }
      }
      if (rep == 1)
          printf("dbg=%u routed=%2d shared=%d stages=%u: %.1f us/launch, %.1f MB, %.0f GB/s (incl memset) SB=%u\n", dbg, n_routed, shared,
                 fl.stages, ms * 1e3 / iters, bytes / 1e6, bytes / (ms * 1e-3 / iters) / 1e9, fl.stage_bytes);
      }
    }
  }
  return 0;
}
