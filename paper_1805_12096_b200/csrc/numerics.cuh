// numerics.cuh — the arithmetic contract every kernel follows (R1-R6, R20).
//
//   Q(x)      = RNE(clip(x, +-c) * sigma), fp32 multiply        (R1, R2)
//   lin       = fmaf((float)acc, s, b) with exact s32 acc        (R3, R5)
//   sigmoid   = fp64 1/(1+exp(-x)) rounded once                  (R20)
//   LN / attention reductions in fp64, one rounding to fp32      (R20)
//   elementwise fp32 ops are single IEEE ops: explicit __f*_rn intrinsics and
//   the whole library is compiled with -fmad=false, so nothing is contracted.
#pragma once
#include <cstdint>

namespace mnmt {

__device__ __forceinline__ int32_t q8(float x, float clip, float sigma) {
  float v = fminf(fmaxf(x, -clip), clip);
  return __float2int_rn(__fmul_rn(v, sigma));
}

__device__ __forceinline__ float dequant(int32_t acc, float s, float b) {
  return __fmaf_rn(__int2float_rn(acc), s, b);
}

__device__ __forceinline__ float sigmoid_f64(float x) {
  return (float)(1.0 / (1.0 + exp(-(double)x)));
}

__device__ __forceinline__ float relu(float x) { return x > 0.0f ? x : 0.0f; }

// Order-preserving map float -> u32 (larger float => larger key); -0 == +0.
__device__ __forceinline__ uint32_t float_order_key(float f) {
  if (f == 0.0f) f = 0.0f;
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// Packed argmax key: max logit wins; among equal logits the LOWEST column wins (R15).
__device__ __forceinline__ unsigned long long argmax_key(float logit, uint32_t col) {
  return ((unsigned long long)float_order_key(logit) << 32) | (unsigned long long)(0xFFFFFFFFu - col);
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace mnmt
