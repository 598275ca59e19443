// The one f64 summation order of a token's predictor logit (predictor.py:76,
// z_t = q . x_t accumulated in f64, kernels.py:41-54), shared by the FFN-input
// RMSNorm (norm.cu, fused logits) and the predictor's own first pooling pass
// (predictor.cu logits_kernel), so both produce bit-identical logits.
//
// A row is owned by one 256-thread CTA.  Thread i owns the float4 groups
// g = i + 256 j of the row (j ascending) and keeps four independent f64 FMA
// chains, one per lane of the group; the thread's value is (z0 + z1) + (z2 + z3),
// reduced across the warp by an xor butterfly and across the 8 warps in warp
// order.  Every step is a fixed sequence of IEEE f64 operations, so the sum
// does not depend on the grid, the scheduling or which kernel computes it.
#pragma once

#include <cuda_runtime.h>

namespace ffwd {
namespace rowdot {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum over the CTA in warp order (fixed, deterministic); every thread gets the result.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum(v);
  __syncthreads();  // `red` may still be read from a previous call
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) s += red[w];
  return s;
}

// One float4 group's contribution to the four chains.
__device__ __forceinline__ void accumulate(double (&z)[4], const double (&q)[4],
                                           const float (&x)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) z[e] = fma(q[e], static_cast<double>(x[e]), z[e]);
}

__device__ __forceinline__ double thread_value(const double (&z)[4]) {
  return (z[0] + z[1]) + (z[2] + z[3]);
}

}  // namespace rowdot
}  // namespace ffwd
