// K1: the FastForward expert predictor and the per-block top-k.
//
//   K1a pool_kernel      z_t = f32(q . x_t) (f64 accumulate), logits = z / f32(sqrt d)
//                        (IEEE f32 division, predictor.py:76), softmax in f64 -> f32
//                        (kernels.py:57-80), pooled = f32(sum_t p_t x_t) (f64 accumulate).
//   K1b gemm_f64acc      relu(f32(pooled . W1)) and f32(h . W2) (kernels.py:41-54,92-93).
//   K1c topk_kernel      radix select over order-preserving 32-bit keys: descending score,
//                        -0 == +0, NaN after every number, ties -> lower index
//                        (kernels.py:139-149); emits the kept set ascending, optionally
//                        filtered to one tensor-parallel rank's strided neuron shard.
//
// Every product is accumulated in fp64 and rounded once to f32, so scores are
// bit-identical to the reference's and the selected indices are exact.  The
// path is HBM/L2 bound; no tensor cores are involved.
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

constexpr int kPoolThreads = 256;

template <bool kF32>
__global__ void __launch_bounds__(kPoolThreads) pool_kernel(const void* __restrict__ x, int T,
                                                            int d, int blk_begin,
                                                            const float* __restrict__ query,
                                                            float sqrt_d,
                                                            float* __restrict__ pooled) {
  __shared__ float logit[kBlockTokens];
  __shared__ float prob[kBlockTokens];
  const int b = blk_begin + blockIdx.x;
  const int tok0 = b * kBlockTokens;
  const int n = min(kBlockTokens, T - tok0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // -- z_t = q . x_t, one warp per token, f64 accumulation (kernels.py:53)
  for (int t = warp; t < n; t += kPoolThreads / 32) {
    double acc = 0.0;
    const size_t row = static_cast<size_t>(tok0 + t) * d;
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
    if (lane == 0) logit[t] = __fdiv_rn(static_cast<float>(acc), sqrt_d);  // predictor.py:76
  }
  __syncthreads();

  // -- softmax over the block in f64, rounded to f32 (kernels.py:57-80)
  if (warp == 0) {
    double m = -INFINITY;
    for (int t = lane; t < n; t += 32) m = fmax(m, static_cast<double>(logit[t]));
    m = warp_max_f64(m);
    double e[kBlockTokens / 32];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kBlockTokens / 32; ++j) {
      const int t = lane + 32 * j;
      e[j] = t < n ? exp(static_cast<double>(logit[t]) - m) : 0.0;
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

  // -- pooled = f32(sum_t p_t x_t), f64 accumulation
  for (int c = threadIdx.x * 8; c < d; c += kPoolThreads * 8) {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
    for (int t = 0; t < n; ++t) {
      float xv[8];
      load8<kF32>(x, static_cast<size_t>(tok0 + t) * d + c, xv);
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
}

// C[M x N] = f32(A[M x K] . B[K x N]), f64 accumulation, row-major f32 operands;
// optional relu applied after the f32 rounding (relu(matmul(.)) in predictor.py:79).
constexpr int GBM = 32, GBN = 64, GBK = 32, GTHREADS = 128;

__global__ void __launch_bounds__(GTHREADS) gemm_f64acc_kernel(const float* __restrict__ A,
                                                               const float* __restrict__ B,
                                                               float* __restrict__ C, int M,
                                                               int K, int N, int relu) {
  __shared__ double As[GBK][GBM + 1];
  __shared__ double Bs[GBK][GBN];
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int tm = threadIdx.x / 16, tn = threadIdx.x % 16;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  for (int k0 = 0; k0 < K; k0 += GBK) {
    for (int e = threadIdx.x; e < GBM * GBK; e += GTHREADS) {
      const int mm = e / GBK, kk = e % GBK;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? static_cast<double>(A[static_cast<size_t>(gm) * K + gk])
                                      : 0.0;
    }
    for (int e = threadIdx.x; e < GBK * GBN; e += GTHREADS) {
      const int kk = e / GBN, nn = e % GBN;
      const int gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < K && gn < N) ? static_cast<double>(B[static_cast<size_t>(gk) * N + gn])
                                      : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GBK; ++kk) {
      double a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tm * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tn + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bv[j], acc[i][j]);
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
      float v = static_cast<float>(acc[i][j]);
      if (relu) v = fmaxf(v, 0.0f);
      C[static_cast<size_t>(gm) * N + gn] = v;
    }
  }
}

// ------------------------------------------------------------------ top-k
constexpr int kTopkThreads = 1024;

// Order-preserving key: larger key = earlier in np.argsort(-s, kind="stable").
__device__ __forceinline__ uint32_t rank_key(float s) {
  if (isnan(s)) return 0u;  // NaN sorts after every number
  uint32_t u = __float_as_uint(s);
  if (u == 0x80000000u) u = 0u;  // -0.0 ties with +0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Block-wide exclusive scan of one int per thread (1024 threads).
__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int wv = warp_tot[lane];
    int wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    warp_tot[lane] = wi - wv;  // exclusive warp offsets
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const int r = warp_tot[warp] + incl - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kTopkThreads) topk_kernel(
    const float* __restrict__ scores, int f, int k, int tp_rank, int tp_size,
    int32_t* __restrict__ idx_global, int ld_global, int32_t* __restrict__ idx_local,
    int ld_local, int32_t* __restrict__ counts) {
  __shared__ int hist[256];
  __shared__ int warp_tot[32];
  __shared__ int s_total;
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining;
  const float* s = scores + static_cast<size_t>(blockIdx.x) * f;
  const int tid = threadIdx.x;

  uint32_t prefix = 0, pmask = 0;
  int remaining = k;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < f; i += kTopkThreads) {
      const uint32_t key = rank_key(s[i]);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins [255-8l-7, 255-8l]; scan from the top bin down
      int c[8], lsum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - 8 * tid - j];
        lsum += c[j];
      }
      int incl = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += t;
      }
      int above = incl - lsum;  // keys in higher bins than this lane's
      const bool mine = above < remaining && incl >= remaining;
      if (mine) {
        int bin = 255 - 8 * tid, cum = above;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (cum + c[j] >= remaining) {
            bin = 255 - 8 * tid - j;
            break;
          }
          cum += c[j];
        }
        s_prefix = prefix | (static_cast<uint32_t>(bin) << shift);
        s_remaining = remaining - cum;
      }
    }
    __syncthreads();
    prefix = s_prefix;
    remaining = s_remaining;
    pmask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t thr = prefix;  // key of the k-th largest score
  const int need_eq = remaining;  // how many keys == thr to keep (lowest index first)

  // -- compaction in index order: contiguous chunk per thread
  const int per = (f + kTopkThreads - 1) / kTopkThreads;
  const int lo = min(f, tid * per), hi = min(f, lo + per);
  int gt = 0, eq = 0;
  for (int i = lo; i < hi; ++i) {
    const uint32_t key = rank_key(s[i]);
    gt += key > thr;
    eq += key == thr;
  }
  const int eq_before = block_exclusive_scan(eq, warp_tot, &s_total);
  int take_eq = min(eq, max(0, need_eq - eq_before));
  // first pass over the chunk: count kept (global and rank-local)
  int kept = 0, kept_loc = 0;
  {
    int te = take_eq;
    for (int i = lo; i < hi; ++i) {
      const uint32_t key = rank_key(s[i]);
      bool keep = key > thr;
      if (!keep && key == thr && te > 0) {
        keep = true;
        --te;
      }
      if (keep) {
        ++kept;
        kept_loc += (i % tp_size) == tp_rank;
      }
    }
  }
  const int pos = block_exclusive_scan(kept, warp_tot, &s_total);
  const int pos_loc = block_exclusive_scan(kept_loc, warp_tot, &s_total);
  if (tid == kTopkThreads - 1 && counts != nullptr) counts[blockIdx.x] = pos_loc + kept_loc;
  int p = pos, pl = pos_loc, te = take_eq;
  for (int i = lo; i < hi; ++i) {
    const uint32_t key = rank_key(s[i]);
    bool keep = key > thr;
    if (!keep && key == thr && te > 0) {
      keep = true;
      --te;
    }
    if (!keep) continue;
    if (idx_global) idx_global[static_cast<size_t>(blockIdx.x) * ld_global + p] = i;
    ++p;
    if ((i % tp_size) == tp_rank) {
      if (idx_local) idx_local[static_cast<size_t>(blockIdx.x) * ld_local + pl] = i / tp_size;
      ++pl;
    }
  }
}

}  // namespace

cudaError_t launch_pool(const void* x, bool x_is_f32, int T, int d, int blk_begin, int blk_count,
                        const float* query, float sqrt_d, float* pooled, cudaStream_t s) {
  if (blk_count <= 0) return cudaSuccess;
  if (x_is_f32)
    pool_kernel<true><<<blk_count, kPoolThreads, 0, s>>>(x, T, d, blk_begin, query, sqrt_d,
                                                         pooled);
  else
    pool_kernel<false><<<blk_count, kPoolThreads, 0, s>>>(x, T, d, blk_begin, query, sqrt_d,
                                                          pooled);
  return cudaGetLastError();
}

cudaError_t launch_gemm_f64acc(const float* A, const float* B, float* C, int M, int K, int N,
                               bool relu, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  dim3 grid((N + GBN - 1) / GBN, (M + GBM - 1) / GBM);
  gemm_f64acc_kernel<<<grid, GTHREADS, 0, s>>>(A, B, C, M, K, N, relu ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_topk(const float* scores, int n_rows, int f, int k, int tp_rank, int tp_size,
                        int32_t* idx_global, int ld_global, int32_t* idx_local, int ld_local,
                        int32_t* counts, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  topk_kernel<<<n_rows, kTopkThreads, 0, s>>>(scores, f, k, tp_rank, tp_size, idx_global,
                                              ld_global, idx_local, ld_local, counts);
  return cudaGetLastError();
}

}  // namespace ffwd
