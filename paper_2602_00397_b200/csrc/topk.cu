// K1c: per-block top-k over the predictor scores (kernels.py:139-149 topk_indices,
// sparse.py:49-55 build_mask).
//
// One CTA per block row; the row's keys are staged once in shared memory.  Radix
// select over order-preserving 32-bit keys finds the k-th largest key in three passes
// (12 + 12 + 8 bit digits, histograms in shared memory), then
// a block-wide scan compacts the kept set in index order, so the output is
// ascending like np.sort(argsort(-s, kind="stable")[:k]).  Ties go to the lower
// index, -0.0 == +0.0, NaN ranks below every number (NumPy sorts NaN last).
// Under tensor parallelism the same global selection is filtered to one rank's
// strided shard {j : j % tp_size == tp_rank} and written as local ids j / tp_size
// with a per-row count (the ragged per-(block, rank) k the plan kernel consumes).
#include <cuda_runtime.h>

#include <cstdint>

#include "ffwd_internal.h"
#include "launch.cuh"

namespace ffwd {

namespace {

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

// The same scan over 64-bit values (two packed 32-bit counts); no total.
__device__ __forceinline__ unsigned long long block_exclusive_scan64(unsigned long long v,
                                                                     unsigned long long* wtot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long wv = wtot[lane];
    unsigned long long wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    wtot[lane] = wi - wv;
  }
  __syncthreads();
  return wtot[warp] + incl - v;
}

// Radix digits, most significant first: 12 + 12 + 8 bits.  A 12-bit first digit
// spreads scores of similar magnitude (same sign and exponent) over many bins, which
// keeps the shared-memory histogram atomics nearly conflict free.
__host__ __device__ constexpr int digit_bits(int pass) { return pass == 2 ? 8 : 12; }
__host__ __device__ constexpr int digit_shift(int pass) { return pass == 0 ? 20 : (pass == 1 ? 8 : 0); }
constexpr int kBins = 4096;
constexpr int kBinsPerThread = kBins / kTopkThreads;  // 4

// kCached: the row's keys are staged once in shared memory (f * 4 bytes), else every
// pass re-reads the scores (from L2) -- only for very wide rows.
// `mask` (nullable): the row's selection as a bitmask (bit j of word j / 32 = neuron j
// kept), `ld_mask` words per row -- the compact form the sequence-parallel predictor
// all-gathers between tensor-parallel ranks (tp.SeqParallelTP).
template <bool kCached>
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(
    const float* __restrict__ scores, int f, int k, int tp_rank, int tp_size,
    int32_t* __restrict__ idx_global, int ld_global, int32_t* __restrict__ idx_local,
    int ld_local, int32_t* __restrict__ counts, uint32_t* __restrict__ mask, int ld_mask) {
  extern __shared__ uint32_t s_keys[];
  // two histograms: pass 1 builds hist[1] while pass 0's is still being searched, and
  // pass 2 reuses hist[0] (zeroed during pass 1), so no pass waits on a separate zeroing
  __shared__ __align__(16) int hist[2][kBins];
  __shared__ int warp_tot[32];
  __shared__ unsigned long long warp_tot64[32];
  __shared__ int s_total;
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    int4* h4 = reinterpret_cast<int4*>(&hist[0][0]);
    for (int i = tid; i < 2 * kBins / 4; i += kTopkThreads) h4[i] = make_int4(0, 0, 0, 0);
  }
  pdl_wait();
  pdl_trigger();
  const float* s = scores + static_cast<size_t>(blockIdx.x) * f;
  auto key_at = [&](int i) -> uint32_t {
    if constexpr (kCached) return s_keys[i];
    else return rank_key(__ldg(s + i));
  };
  __syncthreads();
  if constexpr (kCached) {
    // the first pass's histogram (top 12 bits, every key counts) is built while staging
    auto stage = [&](int i, uint32_t key) {
      s_keys[i] = key;
      atomicAdd(&hist[0][key >> digit_shift(0)], 1);
    };
    if ((f & 3) == 0) {
      // four 16 B loads in flight per thread before the first histogram atomic
      const float4* s4 = reinterpret_cast<const float4*>(s);
      const int n4 = f / 4;
      for (int i0 = tid; i0 < n4; i0 += 4 * kTopkThreads) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u * kTopkThreads < n4) v[u] = __ldg(s4 + i0 + u * kTopkThreads);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kTopkThreads;
          if (i >= n4) break;
          stage(4 * i, rank_key(v[u].x));
          stage(4 * i + 1, rank_key(v[u].y));
          stage(4 * i + 2, rank_key(v[u].z));
          stage(4 * i + 3, rank_key(v[u].w));
        }
      }
    } else {
      for (int i = tid; i < f; i += kTopkThreads) stage(i, rank_key(__ldg(s + i)));
    }
  }

  uint32_t prefix = 0, pmask = 0;
  int remaining = k;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = digit_shift(pass);
    const int nb = 1 << digit_bits(pass);
    int* h = hist[pass & 1];
    if (pass == 1)  // pass 2's histogram: hist[0] was last read before the previous barrier
      for (int i = tid; i < (1 << digit_bits(2)); i += kTopkThreads) hist[0][i] = 0;
    if (!kCached || pass > 0) {  // cached: pass 0's histogram came with the staging
      for (int i = tid; i < f; i += kTopkThreads) {
        const uint32_t key = key_at(i);
        if ((key & pmask) == prefix) atomicAdd(&h[(key >> shift) & (nb - 1)], 1);
      }
    }
    __syncthreads();
    // warp w owns bins [nb-1-bpw w-(bpw-1), nb-1-bpw w] in descending order, bpl per lane;
    // warp totals are scanned by every warp, and only the warp holding the
    // remaining-th largest key scans its lanes -- two barriers per pass
    const int bpw = nb / 32;
    const int bpl = bpw >= 32 ? bpw / 32 : 1;
    const int top = nb - 1 - bpw * warp - bpl * lane;
    const bool lane_on = bpl * lane < bpw;
    int c[kBinsPerThread], lsum = 0;
#pragma unroll
    for (int j = 0; j < kBinsPerThread; ++j) {
      c[j] = (lane_on && j < bpl) ? h[top - j] : 0;
      lsum += c[j];
    }
    int incl = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    const int wt = warp_tot[lane];
    int winc = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, winc, o);
      if (lane >= o) winc += t;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, winc >= remaining);
    const int wb = hit ? __ffs(hit) - 1 : 31;
    const int above_w = __shfl_sync(0xffffffffu, winc - wt, wb);
    if (warp == wb) {
      const int above = above_w + incl - lsum;
      if (lane_on && above < remaining && above + lsum >= remaining) {
        int cum = above, bin = top;
#pragma unroll
        for (int j = 0; j < kBinsPerThread; ++j) {
          if (j < bpl && cum + c[j] >= remaining) {
            bin = top - j;
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
    pmask |= static_cast<uint32_t>(nb - 1) << shift;
  }
  const uint32_t thr = prefix;    // key of the k-th largest score
  const int need_eq = remaining;  // how many keys == thr to keep (lowest index first)

  // -- compaction in index order: contiguous chunk per thread.  One pass counts the keys
  // above the threshold and the ties, and one scan of (gt, eq) gives both the tie quota and
  // the output position: the ties taken before thread t are min(need_eq, eq_before).
  const bool tp1 = tp_size == 1;
  const int per = (f + kTopkThreads - 1) / kTopkThreads;
  const int lo = min(f, tid * per), hi = min(f, lo + per);
  int eq = 0, gt = 0;
  for (int i = lo; i < hi; ++i) {
    const uint32_t key = key_at(i);
    eq += key == thr;
    gt += key > thr;
  }
  const unsigned long long before = block_exclusive_scan64(
      (static_cast<unsigned long long>(gt) << 32) | static_cast<unsigned>(eq), warp_tot64);
  const int eq_before = static_cast<int>(before & 0xffffffffu);
  const int gt_before = static_cast<int>(before >> 32);
  const int take_eq = min(eq, max(0, need_eq - eq_before));
  const int kept = gt + take_eq;
  const int pos = gt_before + min(need_eq, eq_before);
  // rank-local count (tensor parallelism only: without it the local list is the global one)
  int kept_loc = kept;
  if (!tp1) {
    kept_loc = 0;
    int te = take_eq;
    for (int i = lo; i < hi; ++i) {
      const uint32_t key = key_at(i);
      bool keep = key > thr;
      if (!keep && key == thr && te > 0) {
        keep = true;
        --te;
      }
      if (keep) kept_loc += (i % tp_size) == tp_rank;
    }
  }
  const int pos_loc = tp1 ? pos : block_exclusive_scan(kept_loc, warp_tot, &s_total);
  if (tid == kTopkThreads - 1 && counts != nullptr) counts[blockIdx.x] = pos_loc + kept_loc;
  const int nw = (f + 31) / 32;
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(&hist[0][0]);  // the histograms are done with
  if (mask) {
    for (int i = tid; i < nw; i += kTopkThreads) s_mask[i] = 0u;
    __syncthreads();
  }
  int p = pos, pl = pos_loc, te = take_eq;
  for (int i = lo; i < hi; ++i) {
    const uint32_t key = key_at(i);
    bool keep = key > thr;
    if (!keep && key == thr && te > 0) {
      keep = true;
      --te;
    }
    if (!keep) continue;
    if (mask) atomicOr(&s_mask[i >> 5], 1u << (i & 31));
    if (idx_global) idx_global[static_cast<size_t>(blockIdx.x) * ld_global + p] = i;
    ++p;
    if (tp1 || (i % tp_size) == tp_rank) {  // tp1: skip the integer divisions
      if (idx_local)
        idx_local[static_cast<size_t>(blockIdx.x) * ld_local + pl] = tp1 ? i : i / tp_size;
      ++pl;
    }
  }
  if (mask) {
    __syncthreads();
    uint32_t* out = mask + static_cast<size_t>(blockIdx.x) * ld_mask;
    for (int i = tid; i < nw; i += kTopkThreads) out[i] = s_mask[i];
  }
}

// One rank's neuron list from a selection bitmask (the sequence-parallel predictor's
// exchange format): row r's local ids u (ascending) with bit tp_rank + tp_size u set, and
// their count -- exactly what topk_kernel writes as idx_local / counts for that rank.
// Thread t owns a contiguous run of "local words" (32 consecutive local ids each, built
// from the strided global bits), so the count is a popcount and the ids come out of the
// set bits in order.
constexpr int kMaskWordsPerThread = 4;
__global__ void __launch_bounds__(kTopkThreads) mask_to_local_kernel(
    const uint32_t* __restrict__ mask, int ld_mask, int f_global, int tp_rank, int tp_size,
    int32_t* __restrict__ idx_local, int ld_local, int32_t* __restrict__ counts) {
  __shared__ int warp_tot[32];
  __shared__ int s_total;
  pdl_wait();
  pdl_trigger();
  const uint32_t* m = mask + static_cast<size_t>(blockIdx.x) * ld_mask;
  const int tid = threadIdx.x;
  const int f_local = (f_global - tp_rank + tp_size - 1) / tp_size;
  const int nlw = (f_local + 31) / 32;
  uint32_t w[kMaskWordsPerThread];
  int n = 0;
#pragma unroll
  for (int q = 0; q < kMaskWordsPerThread; ++q) {
    const int lw = tid * kMaskWordsPerThread + q;
    uint32_t v = 0;
    if (lw < nlw) {
      if (tp_size == 1) {
        v = __ldg(m + lw);
      } else {
        for (int i = 0; i < 32; ++i) {
          const int u = 32 * lw + i;
          if (u >= f_local) break;
          const int j = tp_rank + tp_size * u;
          v |= ((__ldg(m + (j >> 5)) >> (j & 31)) & 1u) << i;
        }
      }
      if (32 * lw + 32 > f_local) v &= (f_local - 32 * lw >= 32) ? ~0u : ((1u << (f_local - 32 * lw)) - 1u);
    }
    w[q] = v;
    n += __popc(v);
  }
  int p = block_exclusive_scan(n, warp_tot, &s_total);
  if (tid == kTopkThreads - 1 && counts) counts[blockIdx.x] = p + n;
  int32_t* out = idx_local + static_cast<size_t>(blockIdx.x) * ld_local;
#pragma unroll
  for (int q = 0; q < kMaskWordsPerThread; ++q) {
    uint32_t v = w[q];
    const int base = 32 * (tid * kMaskWordsPerThread + q);
    while (v) {
      const int i = __ffs(v) - 1;
      out[p++] = base + i;
      v &= v - 1;
    }
  }
}

constexpr size_t kTopkMaxSmem = 190 * 1024;  // + 33 KiB of static histograms

}  // namespace

cudaError_t launch_topk(const float* scores, int n_rows, int f, int k, int tp_rank, int tp_size,
                        int32_t* idx_global, int ld_global, int32_t* idx_local, int ld_local,
                        int32_t* counts, cudaStream_t s, uint32_t* mask, int ld_mask) {
  if (mask && (f + 31) / 32 > kBins) return cudaErrorInvalidValue;
  if (n_rows <= 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(f) * sizeof(uint32_t);
  if (smem <= kTopkMaxSmem) {
    static std::atomic<uint64_t> attr{0};
    if (cudaError_t e = ensure_smem_limit(topk_kernel<true>, kTopkMaxSmem, attr);
        e != cudaSuccess)
      return e;
    return launch_k(topk_kernel<true>, dim3(n_rows), dim3(kTopkThreads), smem, s, 1, scores, f,
                    k, tp_rank, tp_size, idx_global, ld_global, idx_local, ld_local, counts, mask,
                    ld_mask);
  } else {
    return launch_k(topk_kernel<false>, dim3(n_rows), dim3(kTopkThreads), 0, s, 1, scores, f,
                    k, tp_rank, tp_size, idx_global, ld_global, idx_local, ld_local, counts, mask,
                    ld_mask);
  }
  return cudaGetLastError();
}

cudaError_t launch_mask_to_local(const uint32_t* mask, int ld_mask, int n_rows, int f_global,
                                 int tp_rank, int tp_size, int32_t* idx_local, int ld_local,
                                 int32_t* counts, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  const int f_local = (f_global - tp_rank + tp_size - 1) / tp_size;
  if ((f_local + 31) / 32 > kTopkThreads * kMaskWordsPerThread) return cudaErrorInvalidValue;
  return launch_k(mask_to_local_kernel, dim3(n_rows), dim3(kTopkThreads), 0, s, 1, mask, ld_mask,
                  f_global, tp_rank, tp_size, idx_local, ld_local, counts);
}

}  // namespace ffwd
