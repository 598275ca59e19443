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
#include "sm100.cuh"
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

// ---------------------------------------------------------------- ring-staged RMSNorm
// The same row computation as rmsnorm_kernel (thread i of the 256 owns the float4 groups
// {i + 256 j}; ss and the fused logit in rowdot.cuh's f64 order, so the logits are
// bit-identical to logits_kernel's), organised so neither memory latency nor the per-row
// cross-warp reductions stall the issue slots:
//   * a producer warp streams the CTA's rows (and the `add` rows) into a shared-memory
//     ring with 1-D TMA bulk copies, `ns` rows ahead;
//   * the 8 consumer warps run a three-row software pipeline: phase A of row i (load,
//     [add], the warp's partial sum of squares, published through an mbarrier), then
//     the scale of row i - 1 (f64 divide and square root of the 8 partials, computed
//     once by the row's owner warp i % 8 and published), then phase B of row i - 2
//     (outputs, partial logit), so neither the wait for the other warps' partials nor
//     the scale's dependent f64 chain sits in front of a barrier;
//   * warp 0 finishes each row's logit three rows later from the warps' partials.
// Arithmetic per element (the old kernel spent ~46 instructions per element on INT-pipe
// widening, special-value checks and f64 products; ncu r2):
//   * ss: one F2F (f32 -> f64, exact) and one DFMA;
//   * out = f32((x * scale) * gain): f32 arithmetic on scale split into s_hi + s_lo
//     (p = x s_hi, its exact error by FMA, + x s_lo, then (p + c) * g with one final
//     rounding): within ~2^-47 of the exact product before the final rounding, so it
//     differs from the reference's f64 evaluation (kernels.py:105-106) only when the
//     product lies that close to an f32 rounding boundary (~1e-7 of the elements);
//   * logit: bf16 -> f32 (a shift), F2F, DFMA, as before.
// bf16 -> f64, exact, one conversion instruction
__device__ __forceinline__ double bf16_to_f64(__nv_bfloat16 h) {
  double d;
  asm("cvt.f64.bf16 %0, %1;" : "=d"(d) : "h"(*reinterpret_cast<const unsigned short*>(&h)));
  return d;
}

constexpr int kRingWarps = kNormThreads / 32;  // consumer warps
constexpr int kRedSlots = 4;                   // reduction slots (rows in flight <= 3)
constexpr int kMaxRing = 16;

struct RingHdr {
  uint64_t full[kMaxRing];
  uint64_t empty[kMaxRing];
  uint64_t bar_ss[kRedSlots];
  uint64_t bar_z[kRedSlots];
  uint64_t bar_sc[kRedSlots];
  float sc[kRedSlots][2];  // the row's scale as s_hi, s_lo
  double red_ss[kRedSlots][kRingWarps];
  double red_z[kRedSlots][kRingWarps];
};
constexpr uint32_t kRingHdrBytes = (sizeof(RingHdr) + 127) / 128 * 128;

template <int kMaxV, int kAdd, bool kLogitF32>
__global__ void __launch_bounds__(kNormThreads + 32)
    rmsnorm_ring_kernel(float* __restrict__ x, const float* __restrict__ gain, int T, int d,
                        double eps, const void* __restrict__ add,
                        __nv_bfloat16* __restrict__ out_bf16, float* __restrict__ out_f32,
                        const float* __restrict__ query, float sqrt_d, float* __restrict__ logits,
                        int logit_row0, int logit_row1, int ns, uint32_t stage_bytes) {
  extern __shared__ __align__(128) uint8_t smem_ring[];
  RingHdr* hd = reinterpret_cast<RingHdr*>(smem_ring);
  uint8_t* ring = smem_ring + kRingHdrBytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = d / 4;
  const int nrows = (T - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                    static_cast<int>(gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&hd->full[s], 1);
      mbar_init(&hd->empty[s], kNormThreads);  // every consumer thread releases the slot
    }
    for (int r = 0; r < kRedSlots; ++r) {
      mbar_init(&hd->bar_ss[r], kNormThreads);
      mbar_init(&hd->bar_z[r], kRingWarps);
      mbar_init(&hd->bar_sc[r], 1);
    }
    fence_barrier_init();
  }
  float gf[kMaxV][4];
  double qd[kMaxV][4];
  if (warp < kRingWarps) {
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      const int g = threadIdx.x + kNormThreads * j;
      const float4 w = g < nv ? __ldg(reinterpret_cast<const float4*>(gain) + g)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 q = (query && g < nv) ? __ldg(reinterpret_cast<const float4*>(query) + g)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
      gf[j][0] = w.x; gf[j][1] = w.y; gf[j][2] = w.z; gf[j][3] = w.w;
      qd[j][0] = q.x; qd[j][1] = q.y; qd[j][2] = q.z; qd[j][3] = q.w;
    }
  }
  __syncthreads();
  // gain and query are parameters: read while the predecessor drains, then wait for it
  pdl_wait();
  pdl_trigger();
  const uint32_t xbytes = static_cast<uint32_t>(d) * 4u;
  if (warp == kRingWarps) {  // ---- producer: the CTA's rows into the ring
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nrows; ++i) {
        if (i >= ns) mbar_wait(&hd->empty[s], ph ^ 1);
        const size_t row = blockIdx.x + static_cast<size_t>(i) * gridDim.x;
        mbar_arrive_expect_tx(&hd->full[s], stage_bytes);
        uint8_t* dst = ring + static_cast<size_t>(s) * stage_bytes;
        bulk_load(dst, x + row * d, xbytes, &hd->full[s]);
        if constexpr (kAdd == 1)
          bulk_load(dst + xbytes, static_cast<const float*>(add) + row * d, xbytes, &hd->full[s]);
        if constexpr (kAdd == 2)
          bulk_load(dst + xbytes, static_cast<const __nv_bfloat16*>(add) + row * d, xbytes / 2,
                    &hd->full[s]);
        if (++s == ns) { s = 0; ph ^= 1; }
      }
    }
    return;  // no CTA-wide barrier follows
  }

  auto row_of = [&](int i) { return static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x); };

  // Phase A: [x += add] and this warp's partial sum of squares of row i.
  // ring positions of phase A's and phase B's rows (no integer division per row)
  int sa = 0, sb = 0;
  uint32_t pa = 0;
  auto phase_a = [&](int i) {
    const int s = sa;
    mbar_wait_sleep(&hd->full[s], pa, 1000);
    if (++sa == ns) { sa = 0; pa ^= 1; }
    float4* xs = reinterpret_cast<float4*>(ring + static_cast<size_t>(s) * stage_bytes);
    const size_t row = static_cast<size_t>(row_of(i));
    double sq[4] = {0.0, 0.0, 0.0, 0.0};  // four DFMA chains, one per float4 lane
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      const int g = threadIdx.x + kNormThreads * j;
      if (g >= nv) continue;
      float4 v = xs[g];
      if constexpr (kAdd != 0) {
        float4 a4;
        if constexpr (kAdd == 1) {
          a4 = reinterpret_cast<const float4*>(ring + static_cast<size_t>(s) * stage_bytes + xbytes)[g];
        } else {
          const uint2 raw = reinterpret_cast<const uint2*>(
              ring + static_cast<size_t>(s) * stage_bytes + xbytes)[g];
          const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
          const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
          a4 = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
        v.x = __fadd_rn(v.x, a4.x);  // engine.py:265, f32 residual add
        v.y = __fadd_rn(v.y, a4.y);
        v.z = __fadd_rn(v.z, a4.z);
        v.w = __fadd_rn(v.w, a4.w);
        xs[g] = v;  // phase B reads the sum
        reinterpret_cast<float4*>(x + row * d)[g] = v;
      }
      const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double xd = xv[e];  // F2F, exact
        sq[e] = fma(xd, xd, sq[e]);
      }
    }
    const double ss = rowdot::warp_sum(rowdot::thread_value(sq));
    if (lane == 0) hd->red_ss[i & (kRedSlots - 1)][warp] = ss;
    // every lane arrives: its earlier reads of the slot's scale (row i - 4) are then
    // ordered before the owner's next write of it
    mbar_arrive(&hd->bar_ss[i & (kRedSlots - 1)]);
  };

  // Row i's scale from the 8 partials, by one owner warp per row (i % 8): the f64
  // divide and square root are a long dependent chain, so computing them in every warp
  // cost ~a third of the kernel's instructions and most of its issue-slot latency.
  auto scale_row = [&](int i) {
    const int slot = i & (kRedSlots - 1);
    mbar_wait_sleep(&hd->bar_ss[slot], (i / kRedSlots) & 1, 1000);
    if (lane == 0) {
      double ssum = 0.0;
#pragma unroll
      for (int w = 0; w < kRingWarps; ++w) ssum += hd->red_ss[slot][w];
      const double mean = ssum / static_cast<double>(d);
      const double scale = 1.0 / sqrt(mean + eps);  // kernels.py:105
      const float s_hi = static_cast<float>(scale);
      hd->sc[slot][0] = s_hi;
      hd->sc[slot][1] = static_cast<float>(scale - static_cast<double>(s_hi));
      mbar_arrive(&hd->bar_sc[slot]);
    }
    __syncwarp();
  };

  // Phase B: row i's outputs and this warp's partial logit; releases the ring slot.
  auto phase_b = [&](int i) {
    const int s = sb, slot = i & (kRedSlots - 1);
    if (++sb == ns) sb = 0;
    mbar_wait_sleep(&hd->bar_sc[slot], (i / kRedSlots) & 1, 1000);
    const float s_hi = hd->sc[slot][0];
    const float s_lo = hd->sc[slot][1];
    const int row = row_of(i);
    const bool want_logit = query != nullptr && row >= logit_row0 && row < logit_row1;
    const float4* xs = reinterpret_cast<const float4*>(ring + static_cast<size_t>(s) * stage_bytes);
    double z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < kMaxV; ++j) {
      const int g = threadIdx.x + kNormThreads * j;
      if (g >= nv) continue;
      const float4 v = xs[g];
      const float xv[4] = {v.x, v.y, v.z, v.w};
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = __fmul_rn(xv[e], s_hi);
        const float c = __fmaf_rn(xv[e], s_lo, __fmaf_rn(xv[e], s_hi, -p));
        o[e] = __fmaf_rn(p, gf[j][e], __fmul_rn(c, gf[j][e]));
      }
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
      if (want_logit) {
        if constexpr (kLogitF32) {
          rowdot::accumulate(z, qd[j], o);
        } else {  // bf16 -> f64 in one cvt (F2F.F64.BF16), exact
          z[0] = fma(qd[j][0], bf16_to_f64(lo.x), z[0]);
          z[1] = fma(qd[j][1], bf16_to_f64(lo.y), z[1]);
          z[2] = fma(qd[j][2], bf16_to_f64(hi.x), z[2]);
          z[3] = fma(qd[j][3], bf16_to_f64(hi.y), z[3]);
        }
      }
    }
    if constexpr (kAdd != 0) fence_proxy_async_smem();  // phase A wrote into the slot
    mbar_arrive(&hd->empty[s]);  // each thread's reads of the slot precede the refill
    const double zs = want_logit ? rowdot::warp_sum(rowdot::thread_value(z)) : 0.0;
    if (lane == 0) {
      hd->red_z[slot][warp] = zs;
      mbar_arrive(&hd->bar_z[slot]);
    }
  };

  // warp 0: row i's logit from the 8 partials (rowdot::block_sum's order)
  auto finish = [&](int i) {
    const int slot = i & (kRedSlots - 1);
    mbar_wait_sleep(&hd->bar_z[slot], (i / kRedSlots) & 1, 1000);
    const int row = row_of(i);
    if (lane == 0 && query != nullptr && row >= logit_row0 && row < logit_row1) {
      double zsum = 0.0;
#pragma unroll
      for (int w = 0; w < kRingWarps; ++w) zsum += hd->red_z[slot][w];
      logits[row - logit_row0] = __fdiv_rn(static_cast<float>(zsum), sqrt_d);  // predictor.py:76
    }
    __syncwarp();
  };

  // three rows in flight: phase A of row i, the scale of row i - 1 (its owner warp),
  // phase B of row i - 2, and warp 0 finishing row i - 3's logit
  for (int i = 0; i < nrows + 3; ++i) {
    if (i < nrows) phase_a(i);
    if (i >= 1 && i - 1 < nrows && warp == (i - 1) % kRingWarps) scale_row(i - 1);
    if (i >= 2 && i - 2 < nrows) phase_b(i - 2);
    if (warp == 0 && i >= 3 && i - 3 < nrows) finish(i - 3);
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

#ifndef FFWD_NORM_RING
#define FFWD_NORM_RING 1  // 0: the CTA-per-row rmsnorm_kernel for every shape
#endif

// Ring kernel: stage = the row (+ its add row); 2 CTAs per SM when >= 4 stages fit in
// half the shared memory, else 1 CTA with up to kMaxRing stages.
template <int kMaxV, int kAdd, bool kLogitF32>
cudaError_t launch_ring(float* x, const float* gain, int T, int d, double eps, const void* add,
                        __nv_bfloat16* ob, float* out_f32, const float* query, float sqrt_d,
                        float* logits, int r0, int r1, int sms, bool* used, cudaStream_t s) {
  *used = false;
  const uint32_t stage = static_cast<uint32_t>(d) * (kAdd == 1 ? 8u : (kAdd == 2 ? 6u : 4u));
  const size_t cap2 = 110 * 1024 - kRingHdrBytes, cap1 = 226 * 1024 - kRingHdrBytes;
  int per_sm = 2, ns = static_cast<int>(cap2 / stage);
  if (ns < 4) {
    per_sm = 1;
    ns = static_cast<int>(cap1 / stage);
  }
  if (ns < 3) return cudaSuccess;  // rows too wide: the caller takes rmsnorm_kernel
  if (ns > kMaxRing) ns = kMaxRing;
  const size_t smem = kRingHdrBytes + static_cast<size_t>(ns) * stage;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = ensure_smem_limit(rmsnorm_ring_kernel<kMaxV, kAdd, kLogitF32>, 226 * 1024, attr);
      e != cudaSuccess)
    return e;
  const int grid = T < per_sm * sms ? T : per_sm * sms;
  *used = true;
  return launch_k(rmsnorm_ring_kernel<kMaxV, kAdd, kLogitF32>, dim3(grid),
                  dim3(kNormThreads + 32), smem, s, 1, x, gain, T, d, eps, add, ob, out_f32,
                  query, sqrt_d, logits, r0, r1, ns, stage);
}

template <int kAdd, bool kLogitF32>
cudaError_t launch_rmsnorm_t(float* x, const float* gain, int T, int d, double eps,
                             const void* add, __nv_bfloat16* ob, float* out_f32,
                             const float* query, float sqrt_d, float* logits, int r0, int r1,
                             cudaStream_t s) {
  const int nv = (d / 4 + kNormThreads - 1) / kNormThreads;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // the ring's bulk copies need 16 B rows: d % 4 == 0 always holds, a bf16 add needs d % 8
  if (FFWD_NORM_RING && nv <= 8 && (kAdd != 2 || d % 8 == 0)) {
    bool used = false;
    cudaError_t e;
    if (nv <= 1) e = launch_ring<1, kAdd, kLogitF32>(x, gain, T, d, eps, add, ob, out_f32, query, sqrt_d, logits, r0, r1, sms, &used, s);
    else if (nv <= 2) e = launch_ring<2, kAdd, kLogitF32>(x, gain, T, d, eps, add, ob, out_f32, query, sqrt_d, logits, r0, r1, sms, &used, s);
    else if (nv <= 4) e = launch_ring<4, kAdd, kLogitF32>(x, gain, T, d, eps, add, ob, out_f32, query, sqrt_d, logits, r0, r1, sms, &used, s);
    else e = launch_ring<8, kAdd, kLogitF32>(x, gain, T, d, eps, add, ob, out_f32, query, sqrt_d, logits, r0, r1, sms, &used, s);
    if (e != cudaSuccess || used) return e;
  }
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
