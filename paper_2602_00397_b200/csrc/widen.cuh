// Exact widening of bf16 / f32 values to f64 with integer ops.
//
// The f64 arithmetic that keeps the predictor scores bit-exact (kernels.py:41-54) widens
// every bf16 / f32 operand with F2F, which issues at ~16 per clock per SM and bounds the
// streaming passes over X (pooled_kernel, the fused logits of the FFN-input RMSNorm).
// For normal numbers the widening is a bit-field move: rebias the exponent (+896) and
// shift the mantissa -- a few INT-pipe instructions at 4x the rate.  Zero, subnormal,
// inf and NaN inputs are detected and take the F2F path instead, so results are exactly
// those of static_cast<double> for every input.
#pragma once

#include <cstdint>

namespace ffwd {
namespace widen {

// true if the bf16 in the low 16 bits of `h` is zero / subnormal / inf / NaN
__device__ __forceinline__ bool bf16_special(uint32_t h) {
  return ((h & 0x7F80u) - 0x80u) > 0x7E80u;  // exponent field 0 or 0xFF
}

// either bf16 half of a packed pair special
__device__ __forceinline__ bool bf16x2_special(uint32_t w) {
  return bf16_special(w) || bf16_special(w >> 16);
}

// bf16 in the low 16 bits (normal number) -> f64, exact
__device__ __forceinline__ double bf16_normal_to_f64(uint32_t h) {
  const uint32_t hi = (((h & 0x7FFFu) << 13) + (896u << 20)) | ((h & 0x8000u) << 16);
  return __hiloint2double(static_cast<int>(hi), 0);
}

// any bf16 -> f64 through F2F (the fallback)
__device__ __forceinline__ double bf16_to_f64_f2f(uint32_t h) {
  return static_cast<double>(__uint_as_float((h & 0xFFFFu) << 16));
}

// true if the f32 bit pattern `u` is zero / subnormal / inf / NaN
__device__ __forceinline__ bool f32_special(uint32_t u) {
  return ((u & 0x7F800000u) - 0x00800000u) > 0x7E800000u;
}

// f32 bit pattern (normal number) -> f64, exact
__device__ __forceinline__ double f32_normal_to_f64(uint32_t u) {
  const uint32_t hi = (((u & 0x7FFFFFFFu) >> 3) + (896u << 20)) | (u & 0x80000000u);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
}

}  // namespace widen
}  // namespace ffwd
