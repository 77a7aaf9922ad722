// weights.cuh — counter-based synthetic weights (bit-reproducible on CPU).
//
// w(seed, tensor, i) = bf16_rne(((2u - 1) * scale)), u = top 24 bits of a
// splitmix64-finalised counter hash / 2^24, scale = float(sqrt(3 / fan_in)).
// oracle/moe_layer_ref.py regenerates any tensor with the same integer
// arithmetic, so the CPU oracle never needs the GPU's copy.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace moeb {

// tensor ids
__host__ __device__ inline uint64_t tid_router(uint32_t layer) { return ((uint64_t)layer << 20) | (0xFFFFull << 4); }
__host__ __device__ inline uint64_t tid_shared(uint32_t layer, uint32_t m) { return ((uint64_t)layer << 20) | (0xFFFEull << 4) | m; }
__host__ __device__ inline uint64_t tid_shared_gate(uint32_t layer) { return ((uint64_t)layer << 20) | (0xFFFDull << 4); }
__host__ __device__ inline uint64_t tid_expert(uint32_t layer, uint32_t e, uint32_t m) { return ((uint64_t)layer << 20) | ((uint64_t)e << 4) | m; }

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t b;
#ifdef __CUDA_ARCH__
  b = __float_as_uint(f);
#else
  __builtin_memcpy(&b, &f, 4);
#endif
  b += 0x7FFFu + ((b >> 16) & 1u);
  return (uint16_t)(b >> 16);
}

__device__ __forceinline__ uint16_t synth_weight(uint64_t seed, uint64_t tensor, uint64_t i, float scale) {
  const uint64_t z = mix64(seed ^ (tensor * 0x9E3779B97F4A7C15ULL) ^ (i * 0xD1B54A32D192ED03ULL));
  const float u = (float)(uint32_t)(z >> 40) * 5.9604644775390625e-08f;  // 2^-24
  const float w = __fmul_rn(__fadd_rn(__fmul_rn(2.0f, u), -1.0f), scale);
  return f32_to_bf16_rne(w);
}

// Fill dst[0..n) with tensor `tensor` elements [offset, offset+n).
__global__ void synth_kernel(uint16_t* __restrict__ dst, uint64_t n, uint64_t seed, uint64_t tensor,
                             uint64_t offset, float scale) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = synth_weight(seed, tensor, offset + i, scale);
}

// The same tensor stored transposed: logical [rows][cols] -> dst [cols][rows]
// (element (r, c), counter index r*cols + c, lands at c*rows + r).
__global__ void synth_t_kernel(uint16_t* __restrict__ dst, uint32_t rows, uint32_t cols, uint64_t seed,
                               uint64_t tensor, float scale) {
  const uint64_t n = (uint64_t)rows * cols;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = p / rows, r = p % rows;
    dst[p] = synth_weight(seed, tensor, r * cols + c, scale);
  }
}

// One expert (or shared expert) in the row-interleaved layout of the batch-1
// split-K FFN: for every intermediate row r, [gate row r | up row r | down
// column r] (3 x d contiguous bf16), i.e. dst[F][3][d]. Element values are
// the logical tensors' (gate/up [F][d], down [d][F]) counter-based weights.
__global__ void synth_rows_kernel(uint16_t* __restrict__ dst, uint32_t F, uint32_t d, uint64_t seed, uint64_t t_gate,
                                  uint64_t t_up, uint64_t t_down, float s_in, float s_down) {
  const uint64_t n = 3ull * F * d;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = p / (3ull * d), m = (p / d) % 3, c = p % d;
    dst[p] = m == 0 ? synth_weight(seed, t_gate, r * d + c, s_in)
           : m == 1 ? synth_weight(seed, t_up, r * d + c, s_in)
                    : synth_weight(seed, t_down, c * F + r, s_down);
  }
}

// One expert (or shared expert) in the UMMA-tiled layout of the batched
// tensor-core FFN (ffn_umma.cuh): 16 KB [128 rows x 64 K] bf16 tiles in the
// SWIZZLE_128B K-major order (row r, 16 B chunk j stored at chunk j ^ (r % 8)
// of its 128 B line), grouped in 32 KB stages:
//   gate_up: [F/128 units][d/64 K-blocks][gate tile | up tile]
//   down:    [d/128 units][F/128 K-pairs][tile kb = 2p | tile kb = 2p + 1]
// Element values are the logical tensors' (gate/up [F][d], down [d][F]).
__host__ __device__ inline void tiled_coords(uint64_t p, uint32_t F, uint32_t d, uint32_t& m, uint64_t& idx) {
  const uint64_t gu = 2ull * F * d;
  const uint64_t q = p < gu ? p : p - gu;
  const uint64_t blk = q / 16384, e = q % 16384;
  const uint32_t half = (uint32_t)(e / 8192), off = (uint32_t)(e % 8192) * 2u;
  const uint32_t r = (off / 1024u) * 8u + (off % 1024u) / 128u;
  const uint32_t k = ((((off % 128u) / 16u) ^ r) & 7u) * 8u + (off % 16u) / 2u;
  if (p < gu) {
    const uint64_t u = blk / (d / 64), kb = blk % (d / 64);
    m = half;  // 0 gate, 1 up
    idx = (u * 128 + r) * d + kb * 64 + k;
  } else {
    const uint64_t mt = blk / (F / 128), kp = blk % (F / 128);
    m = 2;
    idx = (mt * 128 + r) * F + kp * 128 + half * 64 + k;
  }
}
__global__ void synth_tiled_kernel(uint16_t* __restrict__ dst, uint32_t F, uint32_t d, uint64_t seed, uint64_t t_gate,
                                   uint64_t t_up, uint64_t t_down, float s_in, float s_down) {
  const uint64_t n = 3ull * F * d;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t m;
    uint64_t idx;
    tiled_coords(p, F, d, m, idx);
    dst[p] = synth_weight(seed, m == 0 ? t_gate : m == 1 ? t_up : t_down, idx, m == 2 ? s_down : s_in);
  }
}

}  // namespace moeb
