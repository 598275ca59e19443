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
// Spins are bounded (about a second) and trap instead of hanging the GPU.
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
};

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void wait_flags(const unsigned* f, int n, unsigned epoch) {
  for (int q = 0; q < n; ++q) {
    long long spins = 0;
    while (static_cast<int>(ld_acquire_sys(f + q) - epoch) < 0) {
      __nanosleep(64);
      if (++spins > (1ll << 24)) __trap();  // a peer never arrived: fail loudly
    }
  }
}

__global__ void __launch_bounds__(kArThreads) allreduce_residual_kernel(ArArgs a) {
  const int n = a.n, r = a.rank;
  // ---- arrive: this rank's partial (written by K3 before this kernel) is complete
  if (blockIdx.x == 0 && threadIdx.x < n) {
    __threadfence_system();
    st_release_sys(a.flags[threadIdx.x] + r, a.epoch);
  }
  if (threadIdx.x == 0) wait_flags(a.flags[r], n, a.epoch);
  __syncthreads();

  // ---- reduce my row slice, fused residual add, all-gather stores
  const int r0 = static_cast<int>((static_cast<long long>(a.T) * r) / n);
  const int r1 = static_cast<int>((static_cast<long long>(a.T) * (r + 1)) / n);
  const size_t base = static_cast<size_t>(r0) * a.d;
  const size_t nvec = static_cast<size_t>(r1 - r0) * a.d / 4;  // d % 4 == 0
  for (size_t i = static_cast<size_t>(blockIdx.x) * kArThreads + threadIdx.x; i < nvec;
       i += static_cast<size_t>(gridDim.x) * kArThreads) {
    const size_t e = base + 4 * i;
    float4 s = *reinterpret_cast<const float4*>(a.residual + e);
    for (int p = 0; p < n; ++p) {  // fixed rank order: identical sums on every rank
      const float4 v = __ldcs(reinterpret_cast<const float4*>(a.partial[p] + e));
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    uint2 pk;
    if (a.xnext[0] != nullptr) {
      const __nv_bfloat162 lo = __floats2bfloat162_rn(s.x, s.y);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(s.z, s.w);
      pk.x = *reinterpret_cast<const uint32_t*>(&lo);
      pk.y = *reinterpret_cast<const uint32_t*>(&hi);
    }
    for (int p = 0; p < n; ++p) {
      const int q = (r + p) % n;  // stagger the destinations across ranks
      __stcg(reinterpret_cast<float4*>(a.out[q] + e), s);
      if (a.xnext[0] != nullptr) __stcg(reinterpret_cast<uint2*>(a.xnext[q] + e), pk);
    }
  }

  // ---- depart: the last CTA publishes "rank r's slice is written" on every peer
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
  if (threadIdx.x == 0) wait_flags(a.flags[r] + n, n, a.epoch);
  __syncthreads();
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
  // every CTA spins at the end, so the grid must be co-resident: one wave
  allreduce_residual_kernel<<<max_ctas, kArThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ffwd
