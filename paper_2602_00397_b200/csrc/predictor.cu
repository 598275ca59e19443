// K1a/K1b: the FastForward expert predictor (predictor.py:68-81), fp64-exact.
//
//   logits_kernel   one CTA per token row: logit_t = f32(q . x_t) / f32(sqrt d), the dot
//                   product accumulated in f64 in the fixed order of rowdot.cuh (shared
//                   with the fused RMSNorm producer) and rounded once (kernels.py:41-54),
//                   the divide a true IEEE f32 division (predictor.py:76).
//   pooled_kernel   per (block, 256 columns): p = f32(softmax_f64(logits_b))
//                   (kernels.py:57-80), pooled = f32(sum_t p_t x_t) in f64 (:78).
//                   Runs the blocks in reverse so the rows pass 1 read last hit L2.
//   gemm_f64_kernel relu(f32(pooled . W1)) and f32(h . W2) (predictor.py:79-80) on
//                   the FP64 tensor pipe (DMMA m8n8k4); K split into f64 partials
//                   reduced in fixed order when the output grid cannot fill the GPU.
//
// Every product is accumulated in fp64 and rounded once to f32 exactly where the
// reference rounds, so the scores are bit-identical to it and the selected
// indices exact.  The two pooling passes are HBM bound (X streamed twice, the second
// partly from L2); the GEMMs are FP64 bound (tools/fp64_bench.cu: DMMA 36.9, DFMA
// 33 TFLOP/s on B200).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "ffwd_internal.h"
#include "launch.cuh"

#include <cooperative_groups.h>

// pooled_kernel: 256-column CTAs when the 512-column grid has fewer CTAs than this (0: never)
#ifndef FFWD_POOL_NARROW_BELOW
#define FFWD_POOL_NARROW_BELOW 148
#endif
// pooled_kernel tuning: tokens in flight per lane (bf16) and the CTAs-per-SM register bound
#ifndef FFWD_POOL_BATCH
#define FFWD_POOL_BATCH 8
#endif
#ifndef FFWD_POOL_MINB
#define FFWD_POOL_MINB 3
#endif
#include "rowdot.cuh"
#include "widen.cuh"
#include "sm100.cuh"

namespace ffwd {

namespace cg = cooperative_groups;

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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

// 8 consecutive activations (bf16 or f32) as packed 16 B vectors.
template <bool kF32>
struct Raw8 {
  uint4 v[kF32 ? 2 : 1];
  __device__ __forceinline__ void load(const void* base, size_t elem) {
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const char*>(base) +
                                                    elem * (kF32 ? 4 : 2));
    v[0] = __ldg(p);
    if constexpr (kF32) v[1] = __ldg(p + 1);
  }
  __device__ __forceinline__ void zero() {
    v[0] = make_uint4(0, 0, 0, 0);
    if constexpr (kF32) v[1] = make_uint4(0, 0, 0, 0);
  }
  __device__ __forceinline__ double get(int i) const {  // exact widening of element i
    const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
    if constexpr (kF32) return static_cast<double>(__uint_as_float(w[i]));
    else
      return static_cast<double>(
          __uint_as_float((i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16)));
  }
};

constexpr int kLogitThreads = rowdot::kThreads;
constexpr int kPoolThreads = 256;
constexpr int kPoolCols = 512;   // per CTA: two 256-column warp halves
constexpr int kPoolQuarters = 4; // token quarters of a block

// 4 consecutive activations (bf16 or f32) of a row, widened to f32 (exact).
template <bool kF32>
__device__ __forceinline__ void load4(const void* base, size_t elem, float (&v)[4]) {
  if constexpr (kF32) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(base) + elem));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(
        static_cast<const __nv_bfloat16*>(base) + elem));
    v[0] = __uint_as_float(t.x << 16); v[1] = __uint_as_float(t.x & 0xFFFF0000u);
    v[2] = __uint_as_float(t.y << 16); v[3] = __uint_as_float(t.y & 0xFFFF0000u);
  }
}

// Pass 1: logit_t = f32(q . x_t) / f32(sqrt d) for every token of the predicted blocks
// (predictor.py:76; the matmul accumulates in f64 and rounds once, kernels.py:41-54).
// One 256-thread CTA per row at a time, in the summation order of rowdot.cuh -- the same
// order the fused RMSNorm producer uses, so a logit is bit-identical whichever kernel
// computes it.  Persistent CTAs walk rows with the next row's loads in flight during the
// current row's reduction.  q is widened into registers once per CTA.
template <bool kF32, int kMaxV>
__global__ void __launch_bounds__(kLogitThreads)
    logits_kernel(const void* __restrict__ x, int d, int tok0, int ntok,
                  const float* __restrict__ query, float sqrt_d, float* __restrict__ logits) {
  __shared__ double red[rowdot::kWarps];
  const int nv = d / 4;
  double qd[kMaxV][4];
#pragma unroll
  for (int j = 0; j < kMaxV; ++j) {
    const int g = threadIdx.x + kLogitThreads * j;
    const float4 q = g < nv ? __ldg(reinterpret_cast<const float4*>(query) + g)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    qd[j][0] = q.x; qd[j][1] = q.y; qd[j][2] = q.z; qd[j][3] = q.w;
  }
  pdl_wait();
  pdl_trigger();
  float nxt[kMaxV][4];
  auto load_row = [&](int t) {
    const size_t row = static_cast<size_t>(tok0 + t) * d;
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      const int g = threadIdx.x + kLogitThreads * j;
      if (g < nv) load4<kF32>(x, row + 4 * static_cast<size_t>(g), nxt[j]);
    }
  };
  int t = blockIdx.x;
  if (t < ntok) load_row(t);
  for (; t < ntok; t += gridDim.x) {
    float v[kMaxV][4];
#pragma unroll
    for (int j = 0; j < kMaxV; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) v[j][e] = nxt[j][e];
    if (t + static_cast<int>(gridDim.x) < ntok) load_row(t + gridDim.x);
    double z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      const int g = threadIdx.x + kLogitThreads * j;
      if (g < nv) rowdot::accumulate(z, qd[j], v[j]);
    }
    const double zs = rowdot::block_sum(rowdot::thread_value(z), red);
    if (threadIdx.x == 0) logits[t] = __fdiv_rn(static_cast<float>(zs), sqrt_d);  // predictor.py:76
  }
}

template <bool kF32>
cudaError_t launch_logits(const void* x, int d, int tok0, int ntok, const float* query,
                          float sqrt_d, float* logits, cudaStream_t s) {
  const int nv = (d / 4 + kLogitThreads - 1) / kLogitThreads;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const dim3 grid(std::min(ntok, 8 * sms));
#define FFWD_LOGITS(V)                                                                     \
  return launch_k(logits_kernel<kF32, V>, grid, dim3(kLogitThreads), 0, s, 1, x, d, tok0, ntok, \
                  query, sqrt_d, logits)
  if (nv <= 1) FFWD_LOGITS(1);
  if (nv <= 2) FFWD_LOGITS(2);
  if (nv <= 4) FFWD_LOGITS(4);
  if (nv <= 8) FFWD_LOGITS(8);
  if (nv <= 16) FFWD_LOGITS(16);
#undef FFWD_LOGITS
  return cudaErrorInvalidValue;
}

// Softmax of each block's logits (kernels.py:57-80, non-causal, f64, max-subtracted,
// rounded to f32), once per block: the probabilities the pooling pass weights X with.
// 128 threads = 4 warps of 32 tokens; the sum is the 4 warp butterflies added in order.
__global__ void __launch_bounds__(kBlockTokens)
    softmax_kernel(int T, int blk_begin, const float* __restrict__ logits,
                   float* __restrict__ probs) {
  __shared__ double wred[2][4];
  pdl_wait();
  pdl_trigger();
  const int rel = blockIdx.x;
  const int tok0 = (blk_begin + rel) * kBlockTokens;
  const int n = min(kBlockTokens, T - tok0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double l = threadIdx.x < n ? static_cast<double>(logits[rel * kBlockTokens + threadIdx.x])
                                   : -INFINITY;
  const double wm = warp_max_f64(l);
  if (lane == 0) wred[0][warp] = wm;
  __syncthreads();
  const double m = fmax(fmax(wred[0][0], wred[0][1]), fmax(wred[0][2], wred[0][3]));
  const double e = threadIdx.x < n ? exp(l - m) : 0.0;
  const double ws = warp_sum_f64(e);
  if (lane == 0) wred[1][warp] = ws;
  __syncthreads();
  const double sum = ((wred[1][0] + wred[1][1]) + wred[1][2]) + wred[1][3];
  probs[rel * kBlockTokens + threadIdx.x] = threadIdx.x < n ? static_cast<float>(e / sum) : 0.f;
}

// Pass 2: pooled_b[c] = f32(sum_t p_t x_t[c]) with f64 accumulation (predictor.py:78), p
// from softmax_kernel.  grid (ceil(d / 512), blk_count); blocks run in reverse so the
// rows pass 1 read last are still in L2.  Warp w covers 256 columns (8 per lane, half
// h = w & 1 of the CTA's 512) for the 32 tokens of quarter w >> 1, with kBatch loads of
// 16 B in flight per lane; the four quarter partials are added in order.
// Widening: F2F (bf16 -> f32 is a shift, then one cvt per element) -- the INT-pipe
// widening of r2 cost ~11 instructions per element and made the pass issue bound.
#ifndef FFWD_POOL_F2F
#define FFWD_POOL_F2F 1
#endif
// kHalves = 2: 512 columns per CTA (8 warps); 1: 256 columns (4 warps), for grids under
// one wave (short prompts: twice the CTAs).  Each column's sum is the same either way.
template <bool kF32, int kHalves>
__global__ void __launch_bounds__(kPoolThreads, FFWD_POOL_MINB)
    pooled_kernel(const void* __restrict__ x, int T, int d, int blk_begin, int blk_count,
                  const float* __restrict__ probs, float* __restrict__ pooled) {
  constexpr int kCols = 256 * kHalves;
  constexpr int kThr = 128 * kHalves;
  __shared__ double probd[kBlockTokens];
  __shared__ double red[kPoolQuarters][kCols];
  pdl_wait();
  pdl_trigger();
  const int rel = blk_count - 1 - static_cast<int>(blockIdx.y);
  const int tok0 = (blk_begin + rel) * kBlockTokens;
  const int n = min(kBlockTokens, T - tok0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < kBlockTokens)
    probd[threadIdx.x] = static_cast<double>(probs[rel * kBlockTokens + threadIdx.x]);
  __syncthreads();

  const int half = kHalves == 2 ? warp & 1 : 0, quarter = kHalves == 2 ? warp >> 1 : warp;
  const int cl = half * 256 + lane * 8;  // column within the CTA's kCols
  const int c = blockIdx.x * kCols + cl;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  if (c < d) {
    constexpr int kPer = kBlockTokens / kPoolQuarters;  // 32 tokens per warp
    constexpr int kBatch = kF32 ? FFWD_POOL_BATCH / 2 : FFWD_POOL_BATCH;  // tokens in flight
#pragma unroll 1
    for (int t0 = quarter * kPer; t0 < quarter * kPer + kPer; t0 += kBatch) {
      Raw8<kF32> xr[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        if (t0 + u < n) xr[u].load(x, static_cast<size_t>(tok0 + t0 + u) * d + c);
        else xr[u].zero();
      }
      bool special = false;  // INT-pipe widening unless a lane holds 0/subnormal/inf/NaN
      if constexpr (!kF32 && !FFWD_POOL_F2F) {
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const uint32_t* w = reinterpret_cast<const uint32_t*>(xr[u].v);
#pragma unroll
          for (int q = 0; q < 4; ++q) special |= widen::bf16x2_special(w[q]);
        }
      }
      if (kF32 || FFWD_POOL_F2F || __any_sync(__activemask(), special)) {
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const double pt = probd[t0 + u];
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = fma(pt, xr[u].get(i), acc[i]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const double pt = probd[t0 + u];
          const uint32_t* w = reinterpret_cast<const uint32_t*>(xr[u].v);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            acc[i] = fma(pt, widen::bf16_normal_to_f64(w[i >> 1] >> (16 * (i & 1))), acc[i]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[quarter][cl + i] = acc[i];
  __syncthreads();
  for (int j = threadIdx.x; j < kCols; j += kThr) {
    const int col = blockIdx.x * kCols + j;
    if (col < d) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < kPoolQuarters; ++q) v += red[q][j];
      pooled[static_cast<size_t>(rel) * d + col] = static_cast<float>(v);
    }
  }
}

// Any-shape pooling (predictor.py:68-78 for blocks of `rpb` rows and any d): the drop-in's
// path for shapes the streaming passes above do not take (d % 8 != 0, or one block of
// n > 128 rows).  One CTA per block: per-row logits (warp per row, f64), the f64 softmax
// over the block's n logits (kept in shared memory as f64), then pooled columns with one
// f64 accumulator per thread.  Small shapes only; the prompt path uses the passes above.
template <bool kF32>
__global__ void __launch_bounds__(256)
    pool_generic_kernel(const void* __restrict__ x, int T, int d, int rpb, int blk_begin,
                        const float* __restrict__ query, float sqrt_d,
                        float* __restrict__ pooled) {
  extern __shared__ double sp[];  // [rpb] logits, then probabilities
  __shared__ double wred[32];
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const long long r0 = static_cast<long long>(blk_begin + blockIdx.x) * rpb;
  const int n = static_cast<int>(min(static_cast<long long>(rpb), T - r0));
  auto xat = [&](long long row, int c) -> double {
    const size_t o = static_cast<size_t>(row) * d + c;
    if constexpr (kF32) return static_cast<double>(__ldg(static_cast<const float*>(x) + o));
    else return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(x)[o]));
  };
  for (int t = warp; t < n; t += nw) {
    double a = 0.0;
    for (int c = lane; c < d; c += 32) a = fma(static_cast<double>(__ldg(query + c)), xat(r0 + t, c), a);
    a = warp_sum_f64(a);
    if (lane == 0) sp[t] = static_cast<double>(__fdiv_rn(static_cast<float>(a), sqrt_d));
  }
  __syncthreads();
  double m = -INFINITY;
  for (int t = threadIdx.x; t < n; t += blockDim.x) m = fmax(m, sp[t]);
  m = warp_max_f64(m);
  if (lane == 0) wred[warp] = m;
  __syncthreads();
  m = wred[0];
  for (int w = 1; w < nw; ++w) m = fmax(m, wred[w]);
  __syncthreads();
  double ssum = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const double e = exp(sp[t] - m);
    sp[t] = e;
    ssum += e;
  }
  ssum = warp_sum_f64(ssum);
  if (lane == 0) wred[warp] = ssum;
  __syncthreads();
  double sum = 0.0;
  for (int w = 0; w < nw; ++w) sum += wred[w];
  for (int t = threadIdx.x; t < n; t += blockDim.x)
    sp[t] = static_cast<double>(static_cast<float>(sp[t] / sum));  // f32 probabilities
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < n; ++t) acc = fma(sp[t], xat(r0 + t, c), acc);
    pooled[static_cast<size_t>(blockIdx.x) * d + c] = static_cast<float>(acc);
  }
}

// ------------------------------------------------------------------ f64 GEMM
// C[M x N] = f32(A[M x K] . B[K x N]) (then relu), f32 row-major operands, f64
// accumulation on DMMA m8n8k4.  CTA tile 128 x BN, 4 warps (warp w: rows
// 32w..32w+31, all BN columns); f32 chunks double-buffered in shared memory with
// cp.async and widened to f64 at fragment load.  grid.z > 1 splits K: each split
// writes an f64 partial tile and gemm_reduce_kernel sums them in split order.
constexpr int GBM = 128, GBK = 32, GTHREADS = 128;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int BN>
__global__ void __launch_bounds__(GTHREADS)
    gemm_f64_kernel(const float* __restrict__ A, const float* __restrict__ B,
                    float* __restrict__ C, double* __restrict__ partial, int M, int K, int N,
                    int kper, int relu) {
  constexpr int AP = GBK + 4;  // f32 pitches: fragment loads are bank-conflict free
  constexpr int BP = BN + 8;
  constexpr int NJ = BN / 8;
  __shared__ __align__(16) float As[2][GBM * AP];
  __shared__ __align__(16) float Bs[2][GBK * BP];
  pdl_wait();
  pdl_trigger();
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * BN;
  const int k_lo = blockIdx.z * kper, k_hi = min(K, k_lo + kper);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fc = lane & 3;
  const bool vec = (K & 3) == 0 && (N & 3) == 0;

  auto load_chunk = [&](int buf, int k0) {
    for (int e = threadIdx.x; e < GBM * (GBK / 4); e += GTHREADS) {
      const int r = e / (GBK / 4), c = (e % (GBK / 4)) * 4;
      const int gm = m0 + r, gk = k0 + c;
      float* dst = &As[buf][r * AP + c];
      const float* src = A + static_cast<size_t>(gm) * K + gk;
      if (vec && gm < M && gk + 3 < k_hi) {
        cp_async16(dst, src);
      } else {
        for (int u = 0; u < 4; ++u) dst[u] = (gm < M && gk + u < k_hi) ? __ldg(src + u) : 0.f;
      }
    }
    for (int e = threadIdx.x; e < GBK * (BN / 4); e += GTHREADS) {
      const int r = e / (BN / 4), c = (e % (BN / 4)) * 4;
      const int gk = k0 + r, gn = n0 + c;
      float* dst = &Bs[buf][r * BP + c];
      const float* src = B + static_cast<size_t>(gk) * N + gn;
      if (vec && gk < k_hi && gn + 3 < N) {
        cp_async16(dst, src);
      } else {
        for (int u = 0; u < 4; ++u) dst[u] = (gk < k_hi && gn + u < N) ? __ldg(src + u) : 0.f;
      }
    }
    cp_async_commit();
  };

  double acc[4][NJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  int buf = 0;
  if (k_lo < k_hi) load_chunk(0, k_lo);
  for (int k0 = k_lo; k0 < k_hi; k0 += GBK) {
    if (k0 + GBK < k_hi) {
      load_chunk(buf ^ 1, k0 + GBK);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* as = As[buf];
    const float* bs = Bs[buf];
#pragma unroll
    for (int ks = 0; ks < GBK / 4; ++ks) {
      double a[4], bb[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        a[i] = static_cast<double>(as[(32 * warp + 8 * i + fr) * AP + 4 * ks + fc]);
#pragma unroll
      for (int j = 0; j < NJ; ++j) bb[j] = static_cast<double>(bs[(4 * ks + fc) * BP + 8 * j + fr]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], a[i], bb[j]);
    }
    __syncthreads();
    buf ^= 1;
  }

#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gm = m0 + 32 * warp + 8 * i + fr, gn = n0 + 8 * j + 2 * fc + h;
        if (gm >= M || gn >= N) continue;
        const size_t o = static_cast<size_t>(gm) * N + gn;
        if (partial) {
          partial[static_cast<size_t>(blockIdx.z) * M * N + o] = acc[i][j][h];
        } else {
          float f = static_cast<float>(acc[i][j][h]);
          if (relu) f = fmaxf(f, 0.0f);  // predictor.py:79: relu after the f32 rounding
          C[o] = f;
        }
      }
}

// The scores GEMM (W2: M = predicted blocks <= 128, K = r, N = d_ffn) with A resident:
// each persistent CTA loads h (M x K f32) into shared memory once and streams W2 in
// 16-column tiles, instead of re-reading all of h for every 16 columns.  RG row groups of
// 32 rows (RG = 1 / 2 for M <= 32 / 64) so small M does not pad to 128 rows;
// the 4 warps split as RG row groups x 4/RG column sub-tiles.  Every output element is
// accumulated exactly as in gemm_f64_kernel (same DMMA fragments, same k order), so the
// scores are bit-identical to it.
template <int RG>
__global__ void __launch_bounds__(GTHREADS)
    gemm_f64_resident_kernel(const float* __restrict__ A, const float* __restrict__ B,
                             float* __restrict__ C, int M, int K, int N, int relu) {
  constexpr int CS = 4 / RG;   // 16-column sub-tiles per iteration
  constexpr int CW = 16 * CS;  // columns per iteration
  constexpr int BP = CW + 8;
  extern __shared__ __align__(16) float smf[];
  const int AP = K + 4;
  float* As = smf;                    // [32 RG][AP]
  float* Bs = smf + 32 * RG * AP;     // [2][GBK][BP]
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fc = lane & 3;
  const int rg = warp % RG, cs = warp / RG;
  for (int e = threadIdx.x; e < 32 * RG * (K / 4); e += GTHREADS) {
    const int r = e / (K / 4), c = (e % (K / 4)) * 4;
    float* dst = As + r * AP + c;
    if (r < M) {
      cp_async16(dst, A + static_cast<size_t>(r) * K + c);
    } else {
      dst[0] = dst[1] = dst[2] = dst[3] = 0.f;
    }
  }
  cp_async_commit();
  const int n_tiles = (N + CW - 1) / CW;
  const int nch = K / GBK;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int n0 = t * CW;
    auto load_b = [&](int buf, int k0) {
      for (int e = threadIdx.x; e < GBK * (CW / 4); e += GTHREADS) {
        const int r = e / (CW / 4), c = (e % (CW / 4)) * 4;
        const int gk = k0 + r, gn = n0 + c;
        float* dst = Bs + buf * GBK * BP + r * BP + c;
        const float* src = B + static_cast<size_t>(gk) * N + gn;
        if (gn + 3 < N) {
          cp_async16(dst, src);
        } else {
          for (int u = 0; u < 4; ++u) dst[u] = gn + u < N ? __ldg(src + u) : 0.f;
        }
      }
      cp_async_commit();
    };
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    load_b(0, 0);
    for (int ch = 0; ch < nch; ++ch) {
      const int buf = ch & 1;
      if (ch + 1 < nch) {
        load_b(buf ^ 1, (ch + 1) * GBK);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const float* bs = Bs + buf * GBK * BP;
      const int k0 = ch * GBK;
#pragma unroll
      for (int ks = 0; ks < GBK / 4; ++ks) {
        double a[4], bb[2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          a[i] = static_cast<double>(As[(32 * rg + 8 * i + fr) * AP + k0 + 4 * ks + fc]);
#pragma unroll
        for (int j = 0; j < 2; ++j)
          bb[j] = static_cast<double>(bs[(4 * ks + fc) * BP + 16 * cs + 8 * j + fr]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma(acc[i][j], a[i], bb[j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gm = 32 * rg + 8 * i + fr, gn = n0 + 16 * cs + 8 * j + 2 * fc + h;
          if (gm >= M || gn >= N) continue;
          float f = static_cast<float>(acc[i][j][h]);
          if (relu) f = fmaxf(f, 0.0f);
          C[static_cast<size_t>(gm) * N + gn] = f;
        }
  }
}

// Split-K for short prompts (M <= 64 rows: the 1B shape's W1, a sequence shard's blocks):
// the K splits of one output tile run as one thread-block cluster (grid.x = splits) and
// are summed through distributed shared memory in split order, s = 0 + p_0 + p_1 + ...
// -- the gemm_reduce_kernel order, so no f64 partial round trip through global memory and
// no second launch.  Tiles are 32 RG rows x 32 columns (no padding of 32 rows to 128);
// warp w takes row group w % RG and 8 (RG = 1) or 16 (RG = 2) columns, each element
// accumulated in the same k order as gemm_f64_kernel.
constexpr int kCzBN = 32;
template <int RG>
__global__ void __launch_bounds__(GTHREADS)
    gemm_f64_cluster_kernel(const float* __restrict__ A, const float* __restrict__ B,
                            float* __restrict__ C, int M, int K, int N, int kper, int relu) {
  constexpr int BM = 32 * RG;
  constexpr int AP = GBK + 4;
  constexpr int BP = kCzBN + 8;
  constexpr int WC = kCzBN / (4 / RG);  // columns per warp
  constexpr int NJ = WC / 8;
  // chunk ring: 4 deep for 32-row tiles (a split's K, 4 chunks at the 1B shape, is in
  // flight at once), 2 deep for 64-row tiles (static shared memory)
  constexpr int kNB = RG == 1 ? 4 : 2;
  __shared__ __align__(16) float As[kNB][BM * AP];
  __shared__ __align__(16) float Bs[kNB][GBK * BP];
  __shared__ __align__(16) double part[BM * kCzBN];
  cg::cluster_group cl = cg::this_cluster();
  const int z = static_cast<int>(cl.block_rank()), nz = static_cast<int>(cl.num_blocks());
  pdl_wait();
  pdl_trigger();
  const int n0 = blockIdx.y * kCzBN, m0 = blockIdx.z * BM;
  const int k_lo = z * kper, k_hi = min(K, k_lo + kper);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fc = lane & 3;
  const int rg = warp % RG, wc = (warp / RG) * WC;
  const bool vec = (K & 3) == 0 && (N & 3) == 0;

  auto load_chunk = [&](int buf, int k0) {
    for (int e = threadIdx.x; e < BM * (GBK / 4); e += GTHREADS) {
      const int r = e / (GBK / 4), c = (e % (GBK / 4)) * 4;
      const int gm = m0 + r, gk = k0 + c;
      float* dst = &As[buf][r * AP + c];
      const float* src = A + static_cast<size_t>(gm) * K + gk;
      if (vec && gm < M && gk + 3 < k_hi) {
        cp_async16(dst, src);
      } else {
        for (int u = 0; u < 4; ++u) dst[u] = (gm < M && gk + u < k_hi) ? __ldg(src + u) : 0.f;
      }
    }
    for (int e = threadIdx.x; e < GBK * (kCzBN / 4); e += GTHREADS) {
      const int r = e / (kCzBN / 4), c = (e % (kCzBN / 4)) * 4;
      const int gk = k0 + r, gn = n0 + c;
      float* dst = &Bs[buf][r * BP + c];
      const float* src = B + static_cast<size_t>(gk) * N + gn;
      if (vec && gk < k_hi && gn + 3 < N) {
        cp_async16(dst, src);
      } else {
        for (int u = 0; u < 4; ++u) dst[u] = (gk < k_hi && gn + u < N) ? __ldg(src + u) : 0.f;
      }
    }
    cp_async_commit();
  };

  double acc[4][NJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nch = k_hi > k_lo ? (k_hi - k_lo + GBK - 1) / GBK : 0;
#pragma unroll
  for (int q = 0; q < kNB - 1; ++q) {  // one commit group per chunk slot, empty past the end
    if (q < nch) load_chunk(q, k_lo + q * GBK);
    else cp_async_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    const int nx = ch + kNB - 1;
    if (nx < nch) load_chunk(nx % kNB, k_lo + nx * GBK);
    else cp_async_commit();
    cp_async_wait<kNB - 1>();  // chunk ch has landed
    __syncthreads();
    const float* as = As[ch % kNB];
    const float* bs = Bs[ch % kNB];
#pragma unroll
    for (int ks = 0; ks < GBK / 4; ++ks) {
      double a[4], bb[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        a[i] = static_cast<double>(as[(32 * rg + 8 * i + fr) * AP + 4 * ks + fc]);
#pragma unroll
      for (int j = 0; j < NJ; ++j) bb[j] = static_cast<double>(bs[(4 * ks + fc) * BP + wc + 8 * j + fr]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], a[i], bb[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        part[(32 * rg + 8 * i + fr) * kCzBN + wc + 8 * j + 2 * fc + h] = acc[i][j][h];
  cl.sync();  // every split's partial tile is in its shared memory
  for (int e = z * GTHREADS + threadIdx.x; e < BM * kCzBN; e += nz * GTHREADS) {
    const int gm = m0 + e / kCzBN, gn = n0 + e % kCzBN;
    double s = 0.0;
    for (int q = 0; q < nz; ++q) s += *cl.map_shared_rank(&part[e], q);  // split order
    if (gm < M && gn < N) {
      float v = static_cast<float>(s);
      if (relu) v = fmaxf(v, 0.0f);  // predictor.py:79: relu after the f32 rounding
      C[static_cast<size_t>(gm) * N + gn] = v;
    }
  }
  cl.sync();  // no CTA leaves while its partial tile may still be read
}

__global__ void gemm_reduce_kernel(const double* __restrict__ partial, float* __restrict__ C,
                                   int MN, int splits, int relu) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= MN) return;
  double s = 0.0;
#pragma unroll 8
  for (int z = 0; z < splits; ++z) s += partial[static_cast<size_t>(z) * MN + i];  // fixed order
  float v = static_cast<float>(s);
  if (relu) v = fmaxf(v, 0.0f);
  C[i] = v;
}

// Split-K GEMMs (the W1 layer: few output tiles, long K) use kSplitBN-column tiles and at
// most kMaxSplits K splits.
#ifndef FFWD_SPLIT_BN
#define FFWD_SPLIT_BN 32
#endif
#ifndef FFWD_MAX_SPLITS
#define FFWD_MAX_SPLITS 32
#endif
// h-resident scores GEMM from this many output columns (M <= 64 rows): the 1B shape's
// 32 x 8192 scores take 128 CTAs of 32-row tiles instead of 128-row tiles 3/4 padding
#ifndef FFWD_RESIDENT_MIN_N
#define FFWD_RESIDENT_MIN_N 4096
#endif
constexpr int kResidentMinN = FFWD_RESIDENT_MIN_N;
constexpr int kGemmBN = FFWD_SPLIT_BN;
constexpr int kMaxSplits = FFWD_MAX_SPLITS;

int gemm_splits(int M, int K, int N) {
  const int tiles = ((N + kGemmBN - 1) / kGemmBN) * ((M + GBM - 1) / GBM);
  int splits = 1;
  while (tiles * splits < 2 * 148 && K / (2 * splits) >= 2 * GBK && splits < kMaxSplits)
    splits *= 2;
  return splits;
}

}  // namespace

cudaError_t launch_pool(const void* x, bool x_is_f32, int T, int d, int blk_begin, int blk_count,
                        const float* query, float sqrt_d, float* logits, float* pooled,
                        const float* logits_in, float* probs, cudaStream_t s) {
  if (blk_count <= 0) return cudaSuccess;
  const int tok0 = blk_begin * kBlockTokens;
  const int ntok = std::min(T, (blk_begin + blk_count) * kBlockTokens) - tok0;
  const dim3 g2((d + kPoolCols - 1) / kPoolCols, blk_count);
  // logits_in: precomputed by the producer of X (absolute token index), e.g. the fused
  // RMSNorm; the first pass is then skipped.
  const float* lg = logits_in ? logits_in + tok0 : logits;
  if (!logits_in) {
    cudaError_t e = x_is_f32 ? launch_logits<true>(x, d, tok0, ntok, query, sqrt_d, logits, s)
                             : launch_logits<false>(x, d, tok0, ntok, query, sqrt_d, logits, s);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_k(softmax_kernel, dim3(blk_count), dim3(kBlockTokens), 0, s, 1, T,
                           blk_begin, lg, probs);
  if (e != cudaSuccess) return e;
  const float* pr = probs;
  if (static_cast<long>(g2.x) * g2.y < FFWD_POOL_NARROW_BELOW) {  // under one wave: 256 columns
    const dim3 g1((d + 255) / 256, blk_count);
    if (x_is_f32)
      return launch_k(pooled_kernel<true, 1>, g1, dim3(128), 0, s, 1, x, T, d, blk_begin,
                      blk_count, pr, pooled);
    return launch_k(pooled_kernel<false, 1>, g1, dim3(128), 0, s, 1, x, T, d, blk_begin,
                    blk_count, pr, pooled);
  }
  if (x_is_f32)
    return launch_k(pooled_kernel<true, 2>, g2, dim3(kPoolThreads), 0, s, 1, x, T, d, blk_begin,
                    blk_count, pr, pooled);
  return launch_k(pooled_kernel<false, 2>, g2, dim3(kPoolThreads), 0, s, 1, x, T, d, blk_begin,
                  blk_count, pr, pooled);
}

cudaError_t launch_pool_generic(const void* x, bool x_is_f32, int T, int d, int rpb,
                                int blk_begin, int blk_count, const float* query, float sqrt_d,
                                float* pooled, cudaStream_t s) {
  if (blk_count <= 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(rpb) * sizeof(double);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> a32{0}, a16{0};
  cudaError_t e = x_is_f32 ? ensure_smem_limit(pool_generic_kernel<true>, 200 * 1024, a32)
                           : ensure_smem_limit(pool_generic_kernel<false>, 200 * 1024, a16);
  if (e != cudaSuccess) return e;
  if (x_is_f32)
    return launch_k(pool_generic_kernel<true>, dim3(blk_count), dim3(256), smem, s, 1, x, T, d,
                    rpb, blk_begin, query, sqrt_d, pooled);
  return launch_k(pool_generic_kernel<false>, dim3(blk_count), dim3(256), smem, s, 1, x, T, d,
                  rpb, blk_begin, query, sqrt_d, pooled);
}

cudaError_t launch_logits_only(const void* x, bool x_is_f32, int d, int tok0, int ntok,
                               const float* query, float sqrt_d, float* logits, cudaStream_t s) {
  if (ntok <= 0) return cudaSuccess;
  return x_is_f32 ? launch_logits<true>(x, d, tok0, ntok, query, sqrt_d, logits, s)
                  : launch_logits<false>(x, d, tok0, ntok, query, sqrt_d, logits, s);
}

template <int RG>
cudaError_t launch_resident(const float* A, const float* B, float* C, int M, int K, int N,
                            bool relu, size_t smem, int grid, cudaStream_t s) {
  // one per instantiation: each kernel needs its own.  The limit is raised to the most any
  // call may ask for (200 KiB), not this call's size: the attribute is set only once.
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = ensure_smem_limit(gemm_f64_resident_kernel<RG>, 200 * 1024, attr);
      e != cudaSuccess)
    return e;
  return launch_k(gemm_f64_resident_kernel<RG>, dim3(grid), dim3(GTHREADS), smem, s, 1, A, B, C,
                  M, K, N, relu ? 1 : 0);
}

// The cluster split-K path (gemm_f64_cluster_kernel): M <= 64, at most kCzMax splits.
#ifndef FFWD_CLUSTER_SPLITK
#define FFWD_CLUSTER_SPLITK 1
#endif
constexpr int kCzMax = 16;  // non-portable cluster size (B200 allows 16)
int cluster_splits(int M, int K, int N) {
  if (!FFWD_CLUSTER_SPLITK || M > 64 || N >= kResidentMinN) return 1;
  const int tiles = ((N + kCzBN - 1) / kCzBN) * ((M + 31) / 32);
  int splits = 1;
  while (tiles * splits < 2 * 148 && K / (2 * splits) >= 2 * GBK && splits < kCzMax) splits *= 2;
  return splits;
}

template <int RG>
cudaError_t launch_cluster_splitk(const float* A, const float* B, float* C, int M, int K, int N,
                                  bool relu, int splits, cudaStream_t s) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    if (cudaError_t e = cudaFuncSetAttribute(gemm_f64_cluster_kernel<RG>,
                                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        e != cudaSuccess)
      return e;
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
  const int kper = ((K + splits - 1) / splits + GBK - 1) / GBK * GBK;
  const int z = (K + kper - 1) / kper;
  const dim3 grid(z, (N + kCzBN - 1) / kCzBN, (M + 32 * RG - 1) / (32 * RG));
  return launch_k(gemm_f64_cluster_kernel<RG>, grid, dim3(GTHREADS), 0, s, z, A, B, C, M, K, N,
                  kper, relu ? 1 : 0);
}

int gemm_f64acc_kernels(int M, int K, int N, bool has_partial) {
  if (!has_partial || cluster_splits(M, K, N) > 1) return 1;
  return gemm_splits(M, K, N) > 1 ? 2 : 1;
}

size_t gemm_f64acc_partial_bytes(int M, int K, int N) {
  const int sp = gemm_splits(M, K, N);
  return sp > 1 ? static_cast<size_t>(sp) * M * N * sizeof(double) : 0;
}

cudaError_t launch_gemm_f64acc(const float* A, const float* B, float* C, int M, int K, int N,
                               bool relu, double* partial, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (partial) {
    if (const int cz = cluster_splits(M, K, N); cz > 1) {
      const cudaError_t e = M > 32 ? launch_cluster_splitk<2>(A, B, C, M, K, N, relu, cz, s)
                                   : launch_cluster_splitk<1>(A, B, C, M, K, N, relu, cz, s);
      // a device that cannot co-schedule 16-CTA clusters (e.g. a small MIG slice) rejects
      // the launch synchronously: take the partials + reduce path below instead
      if (e != cudaErrorInvalidClusterSize && e != cudaErrorLaunchOutOfResources) return e;
      (void)cudaGetLastError();
    }
  }
  const int splits = partial ? gemm_splits(M, K, N) : 1;
  const int kper = ((K + splits - 1) / splits + GBK - 1) / GBK * GBK;
  const int z = (K + kper - 1) / kper;
  // Wide outputs (the W2 scores GEMM) take 16-column tiles: twice the CTAs, so more
  // warps per SM keep the DMMA pipe busy.
  // h resident for up to 64 rows (a sequence shard's or a short prompt's blocks); at 128
  // rows the resident tile leaves one 4-warp CTA per SM and runs slower (83 vs 54 us at
  // 8B/16K), so full prompts keep the 16-column tiles below.
  if (N >= kResidentMinN && M <= 64 && K % GBK == 0 && N % 4 == 0) {
    const int rg = M > 32 ? 2 : 1;
    const size_t smem = (static_cast<size_t>(32 * rg) * (K + 4) +
                         2 * GBK * (16 * (4 / rg) + 8)) * sizeof(float);
    if (smem <= 200 * 1024) {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int per_sm = std::max(1, static_cast<int>((220 * 1024) / (smem + 1024)));
      const int tiles = (N + 16 * (4 / rg) - 1) / (16 * (4 / rg));
      const int grid = std::min(tiles, sms * per_sm);
      return rg == 2 ? launch_resident<2>(A, B, C, M, K, N, relu, smem, grid, s)
                     : launch_resident<1>(A, B, C, M, K, N, relu, smem, grid, s);
    }
  }
  if (z == 1 && N >= 16 * 4 * 148) {
    const dim3 g16((N + 15) / 16, (M + GBM - 1) / GBM, 1);
    return launch_k(gemm_f64_kernel<16>, g16, dim3(GTHREADS), 0, s, 1, A, B, C,
                    static_cast<double*>(nullptr), M, K, N, kper, relu ? 1 : 0);
  }
  const dim3 grid((N + kGemmBN - 1) / kGemmBN, (M + GBM - 1) / GBM, z);
  cudaError_t e = launch_k(gemm_f64_kernel<kGemmBN>, grid, dim3(GTHREADS), 0, s, 1, A, B, C,
                           z > 1 ? partial : static_cast<double*>(nullptr), M, K, N, kper,
                           relu ? 1 : 0);
  if (e != cudaSuccess) return e;
  if (z > 1) {
    const int mn = M * N;
    e = launch_k(gemm_reduce_kernel, dim3((mn + 255) / 256), dim3(256), 0, s, 1,
                 static_cast<const double*>(partial), C, mn, z, relu ? 1 : 0);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace ffwd
