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

}  // namespace moeb
