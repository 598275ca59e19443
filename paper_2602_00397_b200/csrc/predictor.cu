// K1a/K1b: the FastForward expert predictor (predictor.py:68-81), fp64-exact.
//
//   logits_kernel   z_t = f32(q . x_t) with f64 accumulation (kernels.py:41-54), then
//                   logit_t = z_t / f32(sqrt d) as a true IEEE f32 division
//                   (predictor.py:76: matmul(...) / np.float32(np.sqrt(d))).
//   pooled_kernel   p = f32(softmax_f64(logits)) (kernels.py:57-80), then
//                   pooled = f32(sum_t p_t x_t) with f64 accumulation (predictor.py:78).
//   gemm_f64acc     relu(f32(pooled . W1)) and f32(h . W2) (predictor.py:79-80),
//                   split-K into f64 partials + a fixed-order reduction when the
//                   output tile grid is too small to fill the GPU.
//
// Every product is accumulated in fp64 and rounded once to f32 exactly where the
// reference rounds, so the scores are bit-identical to it and the selected
// indices exact.  The predictor is HBM / latency bound; no tensor
// cores are involved.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ffwd_internal.h"

namespace ffwd {

namespace {

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Load 8 consecutive activations as f32 (bf16 -> f32 is exact).
template <bool kF32>
__device__ __forceinline__ void load8(const void* base, size_t off, float (&v)[8]) {
  if constexpr (kF32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + off);
    float4 a = __ldg(p), b = __ldg(p + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(
        static_cast<const __nv_bfloat16*>(base) + off));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
}

constexpr int kLogitWarps = 8;        // one warp per token
constexpr int kLogitSlices = kBlockTokens / kLogitWarps;  // CTAs per block
constexpr int kPoolThreads = 64;      // 8 columns per thread -> 512 columns per CTA
constexpr int kPoolCols = kPoolThreads * 8;

// grid (blk_count, kLogitSlices): 8 tokens per CTA, one warp per token.
template <bool kF32>
__global__ void __launch_bounds__(kLogitWarps * 32)
    logits_kernel(const void* __restrict__ x, int T, int d, int blk_begin,
                  const float* __restrict__ query, float sqrt_d, float* __restrict__ logits) {
  const int b = blk_begin + blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.y * kLogitWarps + warp;
  const int tok0 = b * kBlockTokens;
  if (t >= min(kBlockTokens, T - tok0)) return;
  const size_t row = static_cast<size_t>(tok0 + t) * d;
  double acc = 0.0;
  for (int i = lane * 8; i < d; i += 32 * 8) {
    float xv[8];
    load8<kF32>(x, row + i, xv);
    const float4 q0 = __ldg(reinterpret_cast<const float4*>(query + i));
    const float4 q1 = __ldg(reinterpret_cast<const float4*>(query + i) + 1);
    acc = fma(static_cast<double>(q0.x), static_cast<double>(xv[0]), acc);
    acc = fma(static_cast<double>(q0.y), static_cast<double>(xv[1]), acc);
    acc = fma(static_cast<double>(q0.z), static_cast<double>(xv[2]), acc);
    acc = fma(static_cast<double>(q0.w), static_cast<double>(xv[3]), acc);
    acc = fma(static_cast<double>(q1.x), static_cast<double>(xv[4]), acc);
    acc = fma(static_cast<double>(q1.y), static_cast<double>(xv[5]), acc);
    acc = fma(static_cast<double>(q1.z), static_cast<double>(xv[6]), acc);
    acc = fma(static_cast<double>(q1.w), static_cast<double>(xv[7]), acc);
  }
  acc = warp_sum_f64(acc);
  if (lane == 0)
    logits[static_cast<size_t>(blockIdx.x) * kBlockTokens + t] =
        __fdiv_rn(static_cast<float>(acc), sqrt_d);  // predictor.py:76
}

// grid (blk_count, ceil(d / 512)): softmax of the block's logits (every CTA
// recomputes the same 128-wide f64 softmax), then a 512-column slice of pooled.
template <bool kF32>
__global__ void __launch_bounds__(kPoolThreads)
    pooled_kernel(const void* __restrict__ x, int T, int d, int blk_begin,
                  const float* __restrict__ logits, float* __restrict__ pooled) {
  __shared__ float prob[kBlockTokens];
  const int b = blk_begin + blockIdx.x;
  const int tok0 = b * kBlockTokens;
  const int n = min(kBlockTokens, T - tok0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* lg = logits + static_cast<size_t>(blockIdx.x) * kBlockTokens;
  if (warp == 0) {  // kernels.py:57-80 in f64, rounded to f32
    double m = -INFINITY;
    for (int t = lane; t < n; t += 32) m = fmax(m, static_cast<double>(lg[t]));
    m = warp_max_f64(m);
    double e[kBlockTokens / 32];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kBlockTokens / 32; ++j) {
      const int t = lane + 32 * j;
      e[j] = t < n ? exp(static_cast<double>(lg[t]) - m) : 0.0;
      s += e[j];
    }
    s = warp_sum_f64(s);
#pragma unroll
    for (int j = 0; j < kBlockTokens / 32; ++j) {
      const int t = lane + 32 * j;
      if (t < n) prob[t] = static_cast<float>(e[j] / s);
    }
  }
  __syncthreads();
  const int c = blockIdx.y * kPoolCols + threadIdx.x * 8;
  if (c >= d) return;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  const size_t base = static_cast<size_t>(tok0) * d + c;
#pragma unroll 4
  for (int t = 0; t < n; ++t) {
    float xv[8];
    load8<kF32>(x, base + static_cast<size_t>(t) * d, xv);
    const double p = static_cast<double>(prob[t]);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(p, static_cast<double>(xv[i]), acc[i]);
  }
  float4* out = reinterpret_cast<float4*>(pooled + static_cast<size_t>(blockIdx.x) * d + c);
  out[0] = make_float4(static_cast<float>(acc[0]), static_cast<float>(acc[1]),
                       static_cast<float>(acc[2]), static_cast<float>(acc[3]));
  out[1] = make_float4(static_cast<float>(acc[4]), static_cast<float>(acc[5]),
                       static_cast<float>(acc[6]), static_cast<float>(acc[7]));
}

// C[M x N] (+)= A[M x K] . B[K x N], row-major f32 operands, f64 accumulation.
// splits == 1: C = f32(sum) (optionally relu'd after the rounding, predictor.py:79).
// splits > 1:  partial[split][M][N] in f64; gemm_reduce_kernel finishes.
constexpr int GBM = 32, GBN = 64, GBK = 32, GTHREADS = 128;

__global__ void __launch_bounds__(GTHREADS)
    gemm_f64acc_kernel(const float* __restrict__ A, const float* __restrict__ B,
                       float* __restrict__ C, double* __restrict__ partial, int M, int K, int N,
                       int k_per_split, int relu) {
  __shared__ double As[GBK][GBM + 1];
  __shared__ double Bs[GBK][GBN];
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int k_lo = blockIdx.z * k_per_split, k_hi = min(K, k_lo + k_per_split);
  const int tm = threadIdx.x / 16, tn = threadIdx.x % 16;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  for (int k0 = k_lo; k0 < k_hi; k0 += GBK) {
    for (int e = threadIdx.x; e < GBM * GBK; e += GTHREADS) {
      const int mm = e / GBK, kk = e % GBK;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < k_hi)
                       ? static_cast<double>(A[static_cast<size_t>(gm) * K + gk]) : 0.0;
    }
    for (int e = threadIdx.x; e < GBK * GBN; e += GTHREADS) {
      const int kk = e / GBN, nn = e % GBN;
      const int gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < k_hi && gn < N)
                       ? static_cast<double>(B[static_cast<size_t>(gk) * N + gn]) : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GBK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][tm * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tn + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + tm * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tn + 16 * j;
      if (gn >= N) continue;
      if (partial) {
        partial[(static_cast<size_t>(blockIdx.z) * M + gm) * N + gn] = acc[i][j];
      } else {
        float v = static_cast<float>(acc[i][j]);
        if (relu) v = fmaxf(v, 0.0f);
        C[static_cast<size_t>(gm) * N + gn] = v;
      }
    }
  }
}

__global__ void gemm_reduce_kernel(const double* __restrict__ partial, float* __restrict__ C,
                                   int MN, int splits, int relu) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= MN) return;
  double s = 0.0;
  for (int z = 0; z < splits; ++z) s += partial[static_cast<size_t>(z) * MN + i];  // fixed order
  float v = static_cast<float>(s);
  if (relu) v = fmaxf(v, 0.0f);
  C[i] = v;
}

}  // namespace

int gemm_f64acc_splits(int M, int K, int N) {
  if (M <= 0 || N <= 0 || K <= 0) return 1;
  const int tiles = ((N + GBN - 1) / GBN) * ((M + GBM - 1) / GBM);
  int splits = (2 * 148 + tiles - 1) / tiles;
  const int max_splits = (K + GBK - 1) / GBK;
  if (splits > max_splits) splits = max_splits;
  if (splits > 32) splits = 32;
  return splits < 1 ? 1 : splits;
}

size_t gemm_f64acc_partial_bytes(int M, int K, int N) {
  const int s = gemm_f64acc_splits(M, K, N);
  return s > 1 ? static_cast<size_t>(s) * M * N * sizeof(double) : 0;
}

cudaError_t launch_pool(const void* x, bool x_is_f32, int T, int d, int blk_begin, int blk_count,
                        const float* query, float sqrt_d, float* logits, float* pooled,
                        cudaStream_t s) {
  if (blk_count <= 0) return cudaSuccess;
  const dim3 g1(blk_count, kLogitSlices), g2(blk_count, (d + kPoolCols - 1) / kPoolCols);
  if (x_is_f32) {
    logits_kernel<true><<<g1, kLogitWarps * 32, 0, s>>>(x, T, d, blk_begin, query, sqrt_d,
                                                        logits);
    pooled_kernel<true><<<g2, kPoolThreads, 0, s>>>(x, T, d, blk_begin, logits, pooled);
  } else {
    logits_kernel<false><<<g1, kLogitWarps * 32, 0, s>>>(x, T, d, blk_begin, query, sqrt_d,
                                                         logits);
    pooled_kernel<false><<<g2, kPoolThreads, 0, s>>>(x, T, d, blk_begin, logits, pooled);
  }
  return cudaGetLastError();
}

cudaError_t launch_gemm_f64acc(const float* A, const float* B, float* C, int M, int K, int N,
                               bool relu, double* partial, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  const int splits = partial ? gemm_f64acc_splits(M, K, N) : 1;
  const int kps = ((K + splits - 1) / splits + GBK - 1) / GBK * GBK;
  const int z = (K + kps - 1) / kps;
  dim3 grid((N + GBN - 1) / GBN, (M + GBM - 1) / GBM, z);
  gemm_f64acc_kernel<<<grid, GTHREADS, 0, s>>>(A, B, C, z > 1 ? partial : nullptr, M, K, N, kps,
                                               relu ? 1 : 0);
  if (z > 1) {
    const int mn = M * N;
    gemm_reduce_kernel<<<(mn + 255) / 256, 256, 0, s>>>(partial, C, mn, z, relu ? 1 : 0);
  }
  return cudaGetLastError();
}

}  // namespace ffwd
