// Producers of the FFN input on the full-prefill (TTFT) path, engine.py:262-267.
//
//   rmsnorm_kernel  [x += add, the residual add] then
//                   out = f32(x * (1 / sqrt(mean_f64(x^2) + eps)) * gain), all in f64
//                   like kernels.rmsnorm (kernels.py:96-106), written as bf16 (the
//                   FFN / attention GEMM operand) and optionally as f32.  When a
//                   predictor query is given it also emits the predictor logits of
//                   the row (predictor.py:76: f32(q . x) / f32(sqrt d), f64
//                   accumulation) from the bf16 values it just wrote, so the
//                   predictor's first pass over X disappears.
//   rope_kernel     rotary embedding of Q and K in place (engine.py:50-68 apply_rope):
//                   each head's (first half, second half) pairs rotated by the
//                   position angle: f32 storage in f64 from an f64 cos/sin table (one
//                   rounding, bit-exact to the reference); bf16 storage in f32 from f32
//                   copies of the table.
//
// Both are HBM bound: RMSNorm reads 4 B and writes 2 (+4) B per element, RoPE reads
// and writes Q and K once.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "ffwd_internal.h"
#include "launch.cuh"
#include "rowdot.cuh"
#include "widen.cuh"

namespace ffwd {

namespace {

constexpr int kNormThreads = rowdot::kThreads;  // the logit's summation layout (rowdot.cuh)
using rowdot::block_sum;

// Persistent CTAs (2 per SM) walk rows r = blockIdx.x + k gridDim.x; thread i owns the
// float4 groups {i + 256 j} of a row.  The f32 -> f64 widening (F2F, 16 per clock per
// SM) bounds this kernel, so the gain and the predictor query are widened once per CTA
// into registers, each x element once (reused for the square and the output), and the
// next row's loads are issued before the current row's reductions.
// kLogitF32: the logits are dotted with the f32 outputs (the predictor then pools the
// f32 copy, the reference's own f32 FFN input) instead of their bf16 roundings.
template <int kMaxV, int kAdd, bool kLogitF32>
__global__ void __launch_bounds__(kNormThreads, 2)
    rmsnorm_kernel(float* __restrict__ x, const float* __restrict__ gain, int T, int d,
                   double eps, const void* __restrict__ add, __nv_bfloat16* __restrict__ out_bf16,
                   float* __restrict__ out_f32, const float* __restrict__ query, float sqrt_d,
                   float* __restrict__ logits, int logit_row0, int logit_row1) {
  __shared__ double red[kNormThreads / 32];
  const int nv = d / 4;
  double gd[kMaxV][4], qd[kMaxV][4];
#pragma unroll
  for (int j = 0; j < kMaxV; ++j) {
    const int g = threadIdx.x + kNormThreads * j;
    const float4 w = g < nv ? __ldg(reinterpret_cast<const float4*>(gain) + g)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 q = (query && g < nv) ? __ldg(reinterpret_cast<const float4*>(query) + g)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    gd[j][0] = w.x; gd[j][1] = w.y; gd[j][2] = w.z; gd[j][3] = w.w;
    qd[j][0] = q.x; qd[j][1] = q.y; qd[j][2] = q.z; qd[j][3] = q.w;
  }
  // gain and query are parameters, not the predecessor's output: widen them while the
  // predecessor (the previous layer's down projection) drains, then wait for it
  pdl_wait();
  pdl_trigger();
  auto load_row = [&](int row, float4 (&v)[kMaxV]) {
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(row) * d);
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      const int g = threadIdx.x + kNormThreads * j;
      v[j] = g < nv ? xr[g] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float4 nxt[kMaxV];
  int row = blockIdx.x;
  if (row < T) load_row(row, nxt);
  for (; row < T; row += gridDim.x) {
    float4 v[kMaxV];
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) v[j] = nxt[j];
    if (kAdd != 0) {
      float4* xr = reinterpret_cast<float4*>(x + static_cast<size_t>(row) * d);
#pragma unroll
      for (int j = 0; j < kMaxV; ++j) {
        const int g = threadIdx.x + kNormThreads * j;
        if (g >= nv) continue;
        float4 a4;
        if constexpr (kAdd == 1) {
          a4 = __ldg(reinterpret_cast<const float4*>(add) + static_cast<size_t>(row) * nv + g);
        } else {
          const uint2 raw =
              __ldg(reinterpret_cast<const uint2*>(add) + static_cast<size_t>(row) * nv + g);
          const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
          const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
          a4 = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
        v[j].x = __fadd_rn(v[j].x, a4.x);  // engine.py:265, f32 residual add
        v[j].y = __fadd_rn(v[j].y, a4.y);
        v[j].z = __fadd_rn(v[j].z, a4.z);
        v[j].w = __fadd_rn(v[j].w, a4.w);
        xr[g] = v[j];
      }
    }
    if (row + static_cast<int>(gridDim.x) < T) load_row(row + gridDim.x, nxt);  // prefetch
    double xd[kMaxV][4];
    double ss = 0.0;
    bool special = false;  // widen on the INT pipe unless a lane holds 0/subnormal/inf/NaN
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      if (threadIdx.x + kNormThreads * j < nv)
        special |= widen::f32_special(__float_as_uint(v[j].x)) ||
                   widen::f32_special(__float_as_uint(v[j].y)) ||
                   widen::f32_special(__float_as_uint(v[j].z)) ||
                   widen::f32_special(__float_as_uint(v[j].w));
    }
    const bool fast = !__any_sync(0xffffffffu, special);
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      if (fast) {
        xd[j][0] = widen::f32_normal_to_f64(__float_as_uint(v[j].x));
        xd[j][1] = widen::f32_normal_to_f64(__float_as_uint(v[j].y));
        xd[j][2] = widen::f32_normal_to_f64(__float_as_uint(v[j].z));
        xd[j][3] = widen::f32_normal_to_f64(__float_as_uint(v[j].w));
      } else {
        xd[j][0] = v[j].x; xd[j][1] = v[j].y; xd[j][2] = v[j].z; xd[j][3] = v[j].w;
      }
      ss += (xd[j][0] * xd[j][0] + xd[j][1] * xd[j][1]) +
            (xd[j][2] * xd[j][2] + xd[j][3] * xd[j][3]);
    }
    const double mean = block_sum(ss, red) / static_cast<double>(d);
    const double scale = 1.0 / sqrt(mean + eps);  // kernels.py:105
    const bool want_logit = query != nullptr && row >= logit_row0 && row < logit_row1;
    double z[4] = {0.0, 0.0, 0.0, 0.0};  // four independent DFMA chains
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      const int g = threadIdx.x + kNormThreads * j;
      if (g >= nv) continue;
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        o[e] = static_cast<float>(__dmul_rn(__dmul_rn(xd[j][e], scale), gd[j][e]));
      const size_t off = static_cast<size_t>(row) * d + 4 * static_cast<size_t>(g);
      if (out_f32) reinterpret_cast<float4*>(out_f32 + off)[0] = make_float4(o[0], o[1], o[2], o[3]);
      const __nv_bfloat162 lo = __floats2bfloat162_rn(o[0], o[1]);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(o[2], o[3]);
      if (out_bf16) {
        uint2 pk;
        pk.x = *reinterpret_cast<const uint32_t*>(&lo);
        pk.y = *reinterpret_cast<const uint32_t*>(&hi);
        reinterpret_cast<uint2*>(out_bf16 + off)[0] = pk;
      }
      if (want_logit) {  // q . x with x the operand the pooling pass reads
        if constexpr (kLogitF32) {
          rowdot::accumulate(z, qd[j], o);
        } else {
          const uint32_t wl = *reinterpret_cast<const uint32_t*>(&lo);
          const uint32_t wh = *reinterpret_cast<const uint32_t*>(&hi);
          if (!__any_sync(__activemask(),
                          widen::bf16x2_special(wl) || widen::bf16x2_special(wh))) {
            // exact bf16 -> f64 on the INT pipe (same values as the F2F path below)
            z[0] = fma(qd[j][0], widen::bf16_normal_to_f64(wl), z[0]);
            z[1] = fma(qd[j][1], widen::bf16_normal_to_f64(wl >> 16), z[1]);
            z[2] = fma(qd[j][2], widen::bf16_normal_to_f64(wh), z[2]);
            z[3] = fma(qd[j][3], widen::bf16_normal_to_f64(wh >> 16), z[3]);
          } else {
            const float2 l2 = __bfloat1622float2(lo), h2 = __bfloat1622float2(hi);
            const float xb[4] = {l2.x, l2.y, h2.x, h2.y};
            rowdot::accumulate(z, qd[j], xb);
          }
        }
      }
    }
    if (want_logit) {
      const double zs = block_sum(rowdot::thread_value(z), red);
      if (threadIdx.x == 0)
        logits[row - logit_row0] = __fdiv_rn(static_cast<float>(zs), sqrt_d);  // predictor.py:76
    }
  }
}

// One CTA per token; a thread rotates 2 consecutive pairs (i, i+1) of one head at a
// time (vector loads of both halves).  Q heads at column 0, K heads at k_col.
template <typename E>
__global__ void __launch_bounds__(256)
    rope_kernel(E* __restrict__ qk, int row_stride, int k_col, int n_heads, int d_head,
                const double* __restrict__ cos_t, const double* __restrict__ sin_t,
                const float* __restrict__ cos32, const float* __restrict__ sin32, int pos0) {
  using E2 = std::conditional_t<std::is_same_v<E, float>, float2, __nv_bfloat162>;
  const int t = blockIdx.x;
  const int half = d_head / 2;
  const int hu = half / 2;                 // 2-pair units per head
  const int units = 2 * n_heads * hu;      // Q and K
  E* rowp = qk + static_cast<size_t>(t) * row_stride;
  const double* ct = cos_t + static_cast<size_t>(pos0 + t) * half;
  const double* st = sin_t + static_cast<size_t>(pos0 + t) * half;
  for (int u = threadIdx.x; u < units; u += blockDim.x) {
    const int hh = u / hu, i = (u % hu) * 2;
    E* p = rowp + (hh < n_heads ? 0 : k_col) + (hh % n_heads) * d_head;
    E2* p1 = reinterpret_cast<E2*>(p + i);
    E2* p2 = reinterpret_cast<E2*>(p + half + i);
    const E2 a = *p1, b = *p2;
    float a0, a1, b0, b1;
    if constexpr (std::is_same_v<E, float>) {
      a0 = a.x; a1 = a.y; b0 = b.x; b1 = b.y;
    } else {
      const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
      a0 = fa.x; a1 = fa.y; b0 = fb.x; b1 = fb.y;
    }
    float o[4];
    if (cos32 != nullptr) {
      // bf16 storage: f32 arithmetic from f32 tables (the bf16 rounding dominates; F2F-free)
      const float* c32 = cos32 + static_cast<size_t>(pos0 + t) * half;
      const float* s32 = sin32 + static_cast<size_t>(pos0 + t) * half;
      const float xs1[2] = {a0, a1}, xs2[2] = {b0, b1};
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float c = __ldg(c32 + i + e), sn = __ldg(s32 + i + e);
        o[e] = xs1[e] * c - xs2[e] * sn;
        o[2 + e] = xs1[e] * sn + xs2[e] * c;
      }
    } else {
      const double xs1[2] = {a0, a1}, xs2[2] = {b0, b1};
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double c = __ldg(ct + i + e), sn = __ldg(st + i + e);
        // engine.py:65-66, each f64 product and sum rounded separately (no contraction)
        o[e] = static_cast<float>(__dsub_rn(__dmul_rn(xs1[e], c), __dmul_rn(xs2[e], sn)));
        o[2 + e] = static_cast<float>(__dadd_rn(__dmul_rn(xs1[e], sn), __dmul_rn(xs2[e], c)));
      }
    }
    if constexpr (std::is_same_v<E, float>) {
      *p1 = make_float2(o[0], o[1]);
      *p2 = make_float2(o[2], o[3]);
    } else {
      *p1 = __floats2bfloat162_rn(o[0], o[1]);
      *p2 = __floats2bfloat162_rn(o[2], o[3]);
    }
  }
}

}  // namespace

template <int kAdd, bool kLogitF32>
cudaError_t launch_rmsnorm_t(float* x, const float* gain, int T, int d, double eps,
                             const void* add, __nv_bfloat16* ob, float* out_f32,
                             const float* query, float sqrt_d, float* logits, int r0, int r1,
                             cudaStream_t s) {
  const int nv = (d / 4 + kNormThreads - 1) / kNormThreads;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = T < 2 * sms ? T : 2 * sms;
  cudaError_t e = cudaSuccess;
#define FFWD_NORM(V)                                                                       \
  e = launch_k(rmsnorm_kernel<V, kAdd, kLogitF32>, dim3(grid), dim3(kNormThreads), 0, s, 1, x, gain, T, d, \
               eps, add, ob, out_f32, query, sqrt_d, logits, r0, r1)
  if (nv <= 1) FFWD_NORM(1);
  else if (nv <= 2) FFWD_NORM(2);
  else if (nv <= 4) FFWD_NORM(4);
  else if (nv <= 8) FFWD_NORM(8);
  else if (nv <= 16) FFWD_NORM(16);
  else return cudaErrorInvalidValue;
#undef FFWD_NORM
  return e;
}

template <bool kLogitF32>
cudaError_t launch_rmsnorm_l(float* x, const float* gain, int T, int d, double eps,
                             const void* add, int add_kind, __nv_bfloat16* ob, float* out_f32,
                             const float* query, float sqrt_d, float* logits, int logit_row0,
                             int logit_row1, cudaStream_t s) {
  if (add == nullptr || add_kind == 0)
    return launch_rmsnorm_t<0, kLogitF32>(x, gain, T, d, eps, nullptr, ob, out_f32, query, sqrt_d,
                                          logits, logit_row0, logit_row1, s);
  if (add_kind == 1)
    return launch_rmsnorm_t<1, kLogitF32>(x, gain, T, d, eps, add, ob, out_f32, query, sqrt_d,
                                          logits, logit_row0, logit_row1, s);
  return launch_rmsnorm_t<2, kLogitF32>(x, gain, T, d, eps, add, ob, out_f32, query, sqrt_d,
                                        logits, logit_row0, logit_row1, s);
}

cudaError_t launch_rmsnorm(float* x, const float* gain, int T, int d, double eps,
                           const void* add, int add_kind, void* out_bf16, float* out_f32,
                           const float* query, float sqrt_d, float* logits, int logit_row0,
                           int logit_row1, bool logits_from_f32, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  auto* ob = static_cast<__nv_bfloat16*>(out_bf16);
  if (logits_from_f32 && query != nullptr)
    return launch_rmsnorm_l<true>(x, gain, T, d, eps, add, add_kind, ob, out_f32, query, sqrt_d,
                                  logits, logit_row0, logit_row1, s);
  return launch_rmsnorm_l<false>(x, gain, T, d, eps, add, add_kind, ob, out_f32, query, sqrt_d,
                                 logits, logit_row0, logit_row1, s);
}

cudaError_t launch_rope(void* qk, bool is_f32, int T, int row_stride, int k_col, int n_heads,
                        int d_head, const double* cos_t, const double* sin_t, const float* cos32,
                        const float* sin32, int pos0, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  const dim3 grid(T);
  const int units = n_heads * (d_head / 2);  // 2 x n_heads x (d_head / 4)
  const int threads = units >= 256 ? 256 : (units + 31) / 32 * 32;
  if (is_f32)
    rope_kernel<float><<<grid, threads, 0, s>>>(static_cast<float*>(qk), row_stride, k_col,
                                                n_heads, d_head, cos_t, sin_t, nullptr, nullptr,
                                                pos0);
  else
    rope_kernel<__nv_bfloat16><<<grid, threads, 0, s>>>(static_cast<__nv_bfloat16*>(qk),
                                                        row_stride, k_col, n_heads, d_head,
                                                        cos_t, sin_t, cos32, sin32, pos0);
  return cudaGetLastError();
}

}  // namespace ffwd

// ------------------------------------------------------------ hidden column scores
// sparse.hidden_column_scores (sparse.py:94-97): per block b and neuron j,
// f32(sqrt(sum_t h[t][j]^2)) with f64 accumulation over the block's valid tokens.
// H: the bf16 gated activation of the dense up-projection, or any f32 hidden matrix.
namespace ffwd {
namespace {

template <typename E>
__global__ void __launch_bounds__(256)
    hidden_scores_kernel(const E* __restrict__ h, int ld, int T, int f, int rpb,
                         float* __restrict__ scores) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j >= f) return;
  const int t0 = b * rpb, n = min(rpb, T - t0);
  const E* col = h + static_cast<size_t>(t0) * ld + j;
  double s = 0.0;
#pragma unroll 8
  for (int t = 0; t < n; ++t) {
    double v;
    if constexpr (std::is_same_v<E, float>) v = static_cast<double>(col[static_cast<size_t>(t) * ld]);
    else v = static_cast<double>(__bfloat162float(col[static_cast<size_t>(t) * ld]));
    s = fma(v, v, s);
  }
  scores[static_cast<size_t>(b) * f + j] = static_cast<float>(sqrt(s));
}

}  // namespace

cudaError_t launch_hidden_scores(const void* h, bool is_f32, int ld, int T, int f, int rpb,
                                 float* scores, cudaStream_t s) {
  if (rpb <= 0) return cudaErrorInvalidValue;
  const int n_blk = (T + rpb - 1) / rpb;
  if (n_blk <= 0 || f <= 0) return cudaSuccess;
  const dim3 grid((f + 255) / 256, n_blk);
  if (is_f32)
    hidden_scores_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(h), ld, T, f, rpb,
                                                     scores);
  else
    hidden_scores_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(h), ld, T, f, rpb, scores);
  return cudaGetLastError();
}

}  // namespace ffwd
