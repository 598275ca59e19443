// K1a/K1b: the FastForward expert predictor (predictor.py:68-81), fp64-exact.
//
//   pool_kernel     one thread-block cluster per 128-token block; CTA r of the
//                   cluster owns a d/cs column slice of X_b, staged once in shared
//                   memory (X is read from HBM exactly once):
//                     z_t = f32(q . x_t) with f64 accumulation (kernels.py:41-54):
//                         per-slice f64 partials summed across the cluster
//                         through DSMEM in fixed rank order;
//                     logit_t = z_t / f32(sqrt d), a true IEEE f32 division
//                         (predictor.py:76: matmul(...) / np.float32(np.sqrt(d)));
//                     p = f32(softmax_f64(logits)) (kernels.py:57-80);
//                     pooled = f32(sum_t p_t x_t), f64 accumulation (predictor.py:78).
//   gemm_f64_kernel relu(f32(pooled . W1)) and f32(h . W2) (predictor.py:79-80) on
//                   the FP64 tensor pipe (DMMA m8n8k4); K split across a cluster
//                   and reduced through DSMEM in fixed rank order when the output
//                   grid alone cannot fill the GPU.
//
// Every product is accumulated in fp64 and rounded once to f32 exactly where the
// reference rounds, so the scores are bit-identical to it and the selected
// indices exact.  The pool is HBM bound (X once); the GEMMs are FP64 bound
// (tools/fp64_bench.cu: DMMA 36.9, DFMA 33 TFLOP/s on B200).
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "ffwd_internal.h"
#include "sm100.cuh"

namespace cg = cooperative_groups;

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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

// 1-D TMA bulk copy global -> this CTA's shared memory, completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}

__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 8 consecutive activations as f32 (bf16 -> f32 is exact).
template <bool kF32>
__device__ __forceinline__ void load8(const void* p, float (&v)[8]) {
  if constexpr (kF32) {
    const float4 a = reinterpret_cast<const float4*>(p)[0];
    const float4 b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
    const uint4 raw = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
}

constexpr int kPoolThreads = 256;
constexpr size_t kPoolMaxSmem = 72 * 1024;  // 3 CTAs per SM

__host__ __device__ __forceinline__ int pool_slice(int d, int cs) {
  const int w = (d + cs - 1) / cs;
  return (w + 7) / 8 * 8;
}

// grid (cs, blk_count), cluster (cs, 1, 1).  Dynamic shared memory: the CTA's
// query slice widened to f64, then (kCache) its [n x w] slice of X_b with a 16 B
// padded row pitch so per-token row reads are bank-conflict free; otherwise both
// passes read global memory (the second pass hits L2).  The pooled partials of the
// token groups reuse the X area once it is consumed.
template <bool kF32, bool kCache>
__global__ void __launch_bounds__(kPoolThreads, 3)
    pool_kernel(const void* __restrict__ x, int T, int d, int blk_begin,
                const float* __restrict__ query, float sqrt_d, float* __restrict__ pooled) {
  using E = std::conditional_t<kF32, float, __nv_bfloat16>;
  constexpr int kPad = 16 / static_cast<int>(sizeof(E));
  extern __shared__ __align__(16) uint8_t dyn[];
  __shared__ double part2[2][kBlockTokens];
  __shared__ double part[kBlockTokens];
  __shared__ double probd[kBlockTokens];  // f32-rounded softmax, widened once
  __shared__ double wred[2][4];
  __shared__ uint64_t xbar[4];

  cg::cluster_group cluster = cg::this_cluster();
  const int cs = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  const int b = blk_begin + blockIdx.y;
  const int tok0 = b * kBlockTokens;
  const int n = min(kBlockTokens, T - tok0);
  const int w = pool_slice(d, cs);
  const int wp = w + kPad;
  const int c0 = rank * w;
  const int nc = max(0, min(d, c0 + w) - c0);
  const E* xg = static_cast<const E*>(x) + static_cast<size_t>(tok0) * d + c0;
  double* qs = reinterpret_cast<double*>(dyn);
  uint8_t* xs_raw = dyn + static_cast<size_t>(w) * sizeof(double);
  const E* xs = reinterpret_cast<const E*>(xs_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Stage X_b[:, slice] with one TMA bulk copy per row, in 4 groups of 32 rows with
  // their own mbarriers so phase 1 starts on the first rows while the rest land.
  if constexpr (kCache) {
    if (threadIdx.x < 4) mbar_init(&xbar[threadIdx.x], 1);
    fence_barrier_init();
    __syncthreads();
    if (warp == 0 && nc > 0) {
      const uint32_t row_bytes = static_cast<uint32_t>(nc * sizeof(E));
      for (int grp = 0; grp < 4; ++grp) {
        const int rows = max(0, min(32, n - 32 * grp));
        if (lane == 0) mbar_arrive_expect_tx(&xbar[grp], row_bytes * static_cast<uint32_t>(rows));
        __syncwarp();
        const int t = 32 * grp + lane;
        if (lane < rows)
          bulk_g2s(xs_raw + static_cast<size_t>(t) * wp * sizeof(E),
                   xg + static_cast<size_t>(t) * d, row_bytes, &xbar[grp]);
      }
    }
  }
  for (int c = threadIdx.x; c < nc; c += kPoolThreads)
    qs[c] = static_cast<double>(__ldg(query + c0 + c));
  __syncthreads();
  auto row = [&](int t) -> const E* {
    if constexpr (kCache) return xs + static_cast<size_t>(t) * wp;
    else return xg + static_cast<size_t>(t) * d;
  };

  // ---- slice partial of z_t = q . x_t (f64): thread = (token, half of the slice);
  // the query is a shared-memory broadcast, two chains per thread.
  {
    const int t = threadIdx.x % kBlockTokens, h = threadIdx.x / kBlockTokens;
    const int ng = nc / 8, g_lo = h * (ng / 2), g_hi = h ? ng : ng / 2;
    double a0 = 0.0, a1 = 0.0;
    if constexpr (kCache) {
      if (nc > 0) mbar_wait(&xbar[t >> 5], 0);  // this row's group has landed
    }
    if (t < n) {
      const E* xr = row(t);
      for (int g = g_lo; g < g_hi; ++g) {
        float xv[8];
        load8<kF32>(xr + 8 * g, xv);
        const double* q = qs + 8 * g;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a0 = fma(q[i], static_cast<double>(xv[i]), a0);
          a1 = fma(q[4 + i], static_cast<double>(xv[4 + i]), a1);
        }
      }
    }
    part2[h][t] = a0 + a1;
  }
  __syncthreads();
  if (threadIdx.x < kBlockTokens) part[threadIdx.x] = part2[0][threadIdx.x] + part2[1][threadIdx.x];
  cluster.sync();

  // ---- logits (same in every CTA: fixed rank order), softmax over 4 warps
  double l = -INFINITY;
  if (threadIdx.x < n) {
    double z = 0.0;
    for (int r = 0; r < cs; ++r) z += *cluster.map_shared_rank(&part[threadIdx.x], r);
    l = static_cast<double>(__fdiv_rn(static_cast<float>(z), sqrt_d));  // predictor.py:76
  }
  cluster_arrive_release();  // done reading the peers' partials
  const double wm = warp_max_f64(l);  // kernels.py:57-80 in f64, rounded to f32
  if (warp < 4 && lane == 0) wred[0][warp] = wm;
  __syncthreads();
  const double m = fmax(fmax(wred[0][0], wred[0][1]), fmax(wred[0][2], wred[0][3]));
  const double e = threadIdx.x < n ? exp(l - m) : 0.0;
  const double ws = warp_sum_f64(e);
  if (warp < 4 && lane == 0) wred[1][warp] = ws;
  __syncthreads();
  if (threadIdx.x < n) {
    const double sum = ((wred[1][0] + wred[1][1]) + wred[1][2]) + wred[1][3];
    probd[threadIdx.x] = static_cast<double>(static_cast<float>(e / sum));
  }
  __syncthreads();

  // ---- pooled slice: 8 columns per thread x token groups, f64 partials summed in
  // group order (predictor.py:78).
  const int ng = nc / 8;                                       // 8-column groups
  const int cgp = min(kPoolThreads, max(32, (ng + 31) / 32 * 32));  // threads per token group
  const int tgs = kPoolThreads / cgp;                          // token groups
  const int per = (n + tgs - 1) / tgs;
  const int tg = threadIdx.x / cgp;
  double* red = reinterpret_cast<double*>(xs_raw);             // [tgs][cgp * 8] (aliases X)
  for (int g0 = 0; g0 < ng; g0 += cgp) {
    const int g = g0 + threadIdx.x % cgp;
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
    if (tg < tgs && g < ng) {
      const int t_hi = min(n, tg * per + per);
      for (int t = tg * per; t < t_hi; ++t) {
        float xv[8];
        load8<kF32>(row(t) + 8 * g, xv);
        const double pt = probd[t];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(pt, static_cast<double>(xv[i]), acc[i]);
      }
    }
    __syncthreads();  // X (possibly aliased by `red`) fully consumed
    if (tg < tgs)
#pragma unroll
      for (int i = 0; i < 8; ++i) red[tg * cgp * 8 + (threadIdx.x % cgp) * 8 + i] = acc[i];
    __syncthreads();
    for (int c = threadIdx.x; c < min(cgp, ng - g0) * 8; c += kPoolThreads) {
      double v = 0.0;
      for (int q = 0; q < tgs; ++q) v += red[q * cgp * 8 + c];
      pooled[static_cast<size_t>(blockIdx.y) * d + c0 + g0 * 8 + c] = static_cast<float>(v);
    }
    __syncthreads();
  }
  cluster_wait_acquire();  // peers may still be reading `part`
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

__global__ void gemm_reduce_kernel(const double* __restrict__ partial, float* __restrict__ C,
                                   int MN, int splits, int relu) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= MN) return;
  double s = 0.0;
#pragma unroll 8
  for (int z = 0; z < splits; ++z) s += partial[static_cast<size_t>(z) * MN + i];  // fixed order
  float v = static_cast<float>(s);
  if (relu) v = fmaxf(v, 0.0f);
  C[i] = v;
}

constexpr int kGemmBN = 32;

int gemm_splits(int M, int K, int N) {
  const int tiles = ((N + kGemmBN - 1) / kGemmBN) * ((M + GBM - 1) / GBM);
  int splits = 1;
  while (tiles * splits < 2 * 148 && K / (2 * splits) >= 2 * GBK && splits < 32) splits *= 2;
  return splits;
}

int g_pool_cluster = 0;  // resolved on first use: 16 when the device schedules it, else 8

template <bool kF32, bool kCache>
cudaError_t launch_pool_t(const void* x, int T, int d, int blk_begin, int blk_count,
                          const float* query, float sqrt_d, float* pooled, int cs, size_t smem,
                          cudaStream_t s) {
  auto kern = pool_kernel<kF32, kCache>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kPoolMaxSmem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, blk_count, 1);
  cfg.blockDim = dim3(kPoolThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, x, T, d, blk_begin, query, sqrt_d, pooled);
}

}  // namespace

cudaError_t launch_pool(const void* x, bool x_is_f32, int T, int d, int blk_begin, int blk_count,
                        const float* query, float sqrt_d, float* pooled, cudaStream_t s) {
  if (blk_count <= 0) return cudaSuccess;
  if (g_pool_cluster == 0) {
    // Prefer 16-CTA clusters (a 64 KiB bf16 slice per CTA at d = 4096, 2-3 CTAs per
    // SM); fall back to the portable 8 if the device cannot schedule them.
    int n16 = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(kPoolThreads, 1, 1);
    cfg.dynamicSmemBytes = 68 * 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto kern = pool_kernel<false, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kPoolMaxSmem));
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (cudaOccupancyMaxActiveClusters(&n16, kern, &cfg) != cudaSuccess) n16 = 0;
    cudaGetLastError();
    g_pool_cluster = n16 > 0 ? 16 : 8;
  }
  const int cs = d >= 1024 ? g_pool_cluster : 8;
  const int w = pool_slice(d, cs);
  const size_t esz = x_is_f32 ? sizeof(float) : sizeof(__nv_bfloat16);
  const size_t xbytes = static_cast<size_t>(kBlockTokens) * (w + 16 / esz) * esz;
  const size_t qbytes = static_cast<size_t>(w) * sizeof(double);
  const bool cache = qbytes + xbytes <= kPoolMaxSmem;
  const size_t red = kPoolThreads * 8 * sizeof(double);  // pooled partials (alias X)
  const size_t smem = qbytes + (cache ? std::max(xbytes, red) : red);
  if (x_is_f32)
    return cache ? launch_pool_t<true, true>(x, T, d, blk_begin, blk_count, query, sqrt_d, pooled,
                                             cs, smem, s)
                 : launch_pool_t<true, false>(x, T, d, blk_begin, blk_count, query, sqrt_d,
                                              pooled, cs, smem, s);
  return cache ? launch_pool_t<false, true>(x, T, d, blk_begin, blk_count, query, sqrt_d, pooled,
                                            cs, smem, s)
               : launch_pool_t<false, false>(x, T, d, blk_begin, blk_count, query, sqrt_d, pooled,
                                             cs, smem, s);
}

size_t gemm_f64acc_partial_bytes(int M, int K, int N) {
  const int sp = gemm_splits(M, K, N);
  return sp > 1 ? static_cast<size_t>(sp) * M * N * sizeof(double) : 0;
}

cudaError_t launch_gemm_f64acc(const float* A, const float* B, float* C, int M, int K, int N,
                               bool relu, double* partial, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int splits = partial ? gemm_splits(M, K, N) : 1;
  const int kper = ((K + splits - 1) / splits + GBK - 1) / GBK * GBK;
  const int z = (K + kper - 1) / kper;
  // Wide outputs (the W2 scores GEMM) take 16-column tiles: twice the CTAs, so more
  // warps per SM keep the DMMA pipe busy.
  if (z == 1 && N >= 16 * 4 * 148) {
    const dim3 g16((N + 15) / 16, (M + GBM - 1) / GBM, 1);
    gemm_f64_kernel<16><<<g16, GTHREADS, 0, s>>>(A, B, C, nullptr, M, K, N, kper, relu ? 1 : 0);
    return cudaGetLastError();
  }
  const dim3 grid((N + kGemmBN - 1) / kGemmBN, (M + GBM - 1) / GBM, z);
  gemm_f64_kernel<kGemmBN><<<grid, GTHREADS, 0, s>>>(A, B, C, z > 1 ? partial : nullptr, M, K, N,
                                                     kper, relu ? 1 : 0);
  if (z > 1) {
    const int mn = M * N;
    gemm_reduce_kernel<<<(mn + 255) / 256, 256, 0, s>>>(partial, C, mn, z, relu ? 1 : 0);
  }
  return cudaGetLastError();
}

}  // namespace ffwd
