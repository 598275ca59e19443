// Tensor-parallel completion of the down projection over NVLink peer memory
// (one all-reduce of Y per layer after K3), fused with what follows it:
//
//   h_all = residual + sum_p Y_p          (engine.py:308, the residual add)
//   x_next = bf16(h_all)                  (optional: the next layer's FFN input)
//
// One kernel per rank, no NCCL: every rank owns a contiguous row slice, reads that
// slice of every peer's partial Y straight out of the peer's HBM (P2P loads over
// NVLink), adds its own residual rows, and stores the result into every rank's
// output (P2P stores) -- a reduce-scatter and an all-gather in one pass, so the
// partial sums cross NVLink once and no intermediate buffer exists.
//
// Cross-GPU ordering uses per-rank flag words in peer memory with monotonically
// increasing epochs (never reset):
//   arrive   : rank r publishes flags_p[r] = epoch on every peer p after a
//              system-scope fence (its K3 finished earlier in the stream);
//   wait     : every CTA of rank r spins until flags_r[q] >= epoch for all q;
//   depart   : the last CTA of rank r (grid-wide counter) publishes
//              flags_p[N + r] = epoch after all its stores; every CTA then waits for
//              flags_r[N + q] >= epoch, so when the kernel retires on rank r every
//              peer has finished writing rank r's output.
// Spins are bounded by a wall-clock deadline (%globaltimer; ffwd_set_spin_timeout_ms,
// default 60 s, so ordinary rank skew -- first-iteration setup, a host pause -- is
// waited out) and trap instead of hanging the GPU when a peer is really gone.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ffwd_internal.h"

namespace ffwd {

namespace {

constexpr int kArThreads = 512;
constexpr int kMaxRanks = 8;

struct ArArgs {
  const float* partial[kMaxRanks];  // rank p's partial Y (peer pointers)
  float* out[kMaxRanks];            // rank p's residual-stream output
  __nv_bfloat16* xnext[kMaxRanks];  // rank p's next-layer input (nullable)
  unsigned* flags[kMaxRanks];       // rank p's flag words [2N] (+ counter at [2N])
  const float* residual;            // this rank's residual (may alias out[rank])
  int n, rank, T, d;
  unsigned epoch;
  unsigned long long timeout_ns;    // spin deadline per wait
};

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void wait_flags(const unsigned* f, int n, unsigned epoch,
                                           unsigned long long timeout_ns) {
  for (int q = 0; q < n; ++q) {
    const unsigned long long t0 = gtimer_ns();
    while (static_cast<int>(ld_acquire_sys(f + q) - epoch) < 0) {
      __nanosleep(64);
      if (gtimer_ns() - t0 > timeout_ns) __trap();  // a peer never arrived: fail loudly
    }
  }
}

// out_p[rows] = residual[rows] + sum_q partial_q[rows] on every rank p, rows [r0, r1),
// grid-strided over `ctas` CTAs starting at `cta`.  Each thread keeps kUnroll float4 of
// every source in flight (peer loads over NVLink take microseconds: the kernel is bound
// by bytes in flight, not by bandwidth, with one load per thread).
constexpr int kUnroll = 4;

__device__ __forceinline__ void reduce_rows(const ArArgs& a, int r0, int r1, int cta, int ctas) {
  const int n = a.n, r = a.rank;
  const size_t base = static_cast<size_t>(r0) * a.d;
  const size_t nvec = static_cast<size_t>(r1 - r0) * a.d / 4;  // d % 4 == 0
  const size_t stride = static_cast<size_t>(ctas) * kArThreads;
  for (size_t i0 = static_cast<size_t>(cta) * kArThreads + threadIdx.x; i0 < nvec;
       i0 += stride * kUnroll) {
    float4 s[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const size_t i = i0 + u * stride;
      s[u] = i < nvec ? *reinterpret_cast<const float4*>(a.residual + base + 4 * i)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int p = 0; p < n; ++p) {  // fixed rank order: identical sums on every rank
      float4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const size_t i = i0 + u * stride;
        v[u] = i < nvec ? __ldcg(reinterpret_cast<const float4*>(a.partial[p] + base + 4 * i))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        s[u].x += v[u].x;
        s[u].y += v[u].y;
        s[u].z += v[u].z;
        s[u].w += v[u].w;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const size_t i = i0 + u * stride;
      if (i >= nvec) break;
      const size_t e = base + 4 * i;
      uint2 pk;
      if (a.xnext[0] != nullptr) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(s[u].x, s[u].y);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(s[u].z, s[u].w);
        pk.x = *reinterpret_cast<const uint32_t*>(&lo);
        pk.y = *reinterpret_cast<const uint32_t*>(&hi);
      }
      for (int p = 0; p < n; ++p) {
        const int q = (r + p) % n;  // stagger the destinations across ranks
        __stcg(reinterpret_cast<float4*>(a.out[q] + e), s[u]);
        if (a.xnext[0] != nullptr) __stcg(reinterpret_cast<uint2*>(a.xnext[q] + e), pk);
      }
    }
  }
}

// The last CTA of rank r (grid-wide counter) publishes "rank r's rows are written" on
// every peer; every CTA then waits for all peers' departures, so when the kernel retires
// on rank r no peer still reads rank r's partial or writes rank r's output.
__device__ __forceinline__ void depart(const ArArgs& a) {
  const int n = a.n, r = a.rank;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned* ctr = a.flags[r] + 2 * n;
    const unsigned prev = atomicAdd(ctr, 1u);
    last = prev == gridDim.x - 1;
    if (last) atomicExch(ctr, 0u);
  }
  __syncthreads();
  if (last && threadIdx.x < n) st_release_sys(a.flags[threadIdx.x] + n + r, a.epoch);
  if (threadIdx.x == 0) wait_flags(a.flags[r] + n, n, a.epoch, a.timeout_ns);
  __syncthreads();
}

__global__ void __launch_bounds__(kArThreads) allreduce_residual_kernel(ArArgs a) {
  const int n = a.n, r = a.rank;
  // ---- arrive: this rank's partial (written by K3 before this kernel) is complete
  if (blockIdx.x == 0 && threadIdx.x < n) {
    __threadfence_system();
    st_release_sys(a.flags[threadIdx.x] + r, a.epoch);
  }
  if (threadIdx.x == 0) wait_flags(a.flags[r], n, a.epoch, a.timeout_ns);
  __syncthreads();

  // ---- reduce my row slice, fused residual add, all-gather stores
  const int r0 = static_cast<int>((static_cast<long long>(a.T) * r) / n);
  const int r1 = static_cast<int>((static_cast<long long>(a.T) * (r + 1)) / n);
  reduce_rows(a, r0, r1, blockIdx.x, gridDim.x);

  depart(a);
}

// Overlapped with the down projection: the plan's raster order (dense blocks first, then
// the predicted range; plan.cu order_to_block) is the order K3 finishes blocks in, so CTA c
// takes blocks o = c, c + G, ... of that order, waits until every rank's K3 has published
// all column tiles of the block (ydone counters, system-scope release in the K3
// epilogue), and reduces this rank's 1/N of the block's rows -- the transfer of block b
// runs while K3 still computes later blocks.
struct ArOvArgs {
  ArArgs base;
  const unsigned* ydone[kMaxRanks];
  unsigned target;
  int sparse_begin, sparse_count;
};

__global__ void __launch_bounds__(kArThreads) allreduce_overlap_kernel(ArOvArgs ov) {
  const ArArgs& a = ov.base;
  const int n = a.n, r = a.rank;
  const int n_blk = (a.T + kBlockTokens - 1) / kBlockTokens;
  const int n_dense = n_blk - ov.sparse_count;
  for (int o = blockIdx.x; o < n_blk; o += gridDim.x) {
    const int b = o < ov.sparse_begin ? o
                  : o < n_dense      ? ov.sparse_begin + ov.sparse_count + (o - ov.sparse_begin)
                                     : ov.sparse_begin + (o - n_dense);
    if (threadIdx.x == 0) {
      for (int q = 0; q < n; ++q) {
        const unsigned long long t0 = gtimer_ns();
        while (static_cast<int>(ld_acquire_sys(ov.ydone[q] + b) - ov.target) < 0) {
          __nanosleep(128);
          if (gtimer_ns() - t0 > a.timeout_ns) __trap();  // a rank's K3 never finished block b
        }
      }
    }
    __syncthreads();
    const int t0 = b * kBlockTokens;
    const int nt = min(kBlockTokens, a.T - t0);
    reduce_rows(a, t0 + nt * r / n, t0 + nt * (r + 1) / n, 0, 1);
    __syncthreads();
  }
  depart(a);
}

}  // namespace

cudaError_t launch_allreduce_residual(const float* const* partial, float* const* out,
                                      void* const* xnext, unsigned* const* flags, int n,
                                      int rank, const float* residual, int T, int d,
                                      unsigned epoch, int max_ctas, cudaStream_t s) {
  if (n < 1 || n > kMaxRanks) return cudaErrorInvalidValue;
  ArArgs a{};
  for (int p = 0; p < n; ++p) {
    a.partial[p] = partial[p];
    a.out[p] = out[p];
    a.xnext[p] = xnext ? static_cast<__nv_bfloat16*>(xnext[p]) : nullptr;
    a.flags[p] = flags[p];
  }
  a.residual = residual;
  a.n = n;
  a.rank = rank;
  a.T = T;
  a.d = d;
  a.epoch = epoch;
  a.timeout_ns = spin_timeout_ns();
  // every CTA spins at the end, so the grid must be co-resident: one wave
  allreduce_residual_kernel<<<max_ctas, kArThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ffwd

namespace ffwd {

cudaError_t launch_allreduce_overlap(const float* const* partial, float* const* out,
                                     void* const* xnext, unsigned* const* flags,
                                     const unsigned* const* ydone, int n, int rank,
                                     const float* residual, int T, int d, unsigned epoch,
                                     unsigned target, int sparse_begin, int sparse_count,
                                     int max_ctas, cudaStream_t s) {
  if (n < 1 || n > kMaxRanks) return cudaErrorInvalidValue;
  ArOvArgs ov{};
  ArArgs& a = ov.base;
  for (int p = 0; p < n; ++p) {
    a.partial[p] = partial[p];
    a.out[p] = out[p];
    a.xnext[p] = xnext ? static_cast<__nv_bfloat16*>(xnext[p]) : nullptr;
    a.flags[p] = flags[p];
    ov.ydone[p] = ydone[p];
  }
  a.residual = residual;
  a.n = n;
  a.rank = rank;
  a.T = T;
  a.d = d;
  a.epoch = epoch;
  a.timeout_ns = spin_timeout_ns();
  ov.target = target;
  ov.sparse_begin = sparse_begin;
  ov.sparse_count = sparse_count;
  // few CTAs: they spin beside K3 (one K3 CTA per SM leaves room for one of these) and
  // must all be resident for the final departure barrier
  allreduce_overlap_kernel<<<max_ctas, kArThreads, 0, s>>>(ov);
  return cudaGetLastError();
}

}  // namespace ffwd
