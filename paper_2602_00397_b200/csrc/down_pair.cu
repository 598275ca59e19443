// K3 for block pairs: the down projection of the neurons two adjacent blocks both selected,
// as one CTA-pair (tcgen05 cta_group::2) gather-GEMM.
//
//   Y_b[:, n0:n0+256] (+)= H_b[:, 0:s] . W_down[S[0:s], n0:n0+256]     b = b0 (CTA 0), b1 (CTA 1)
//   (sparse.py:91 down matmul over the shared part of the two selections, engine.py:284-300)
//
// The two blocks' index lists start with the same s neurons (S, a multiple of 64), so the
// W_down rows of a stage feed both blocks: CTA r gathers columns [n0 + 128 r, +128) of
// the stage's 64 rows and loads its own block's H tile, and the leader's MMA (M = 256:
// CTA r's A rows are block b_r's tokens; B split along N between the CTAs) accumulates
// both blocks' 128 x 256 tiles, one in each CTA's TMEM.  Per SM and stage that is half the
// gathered bytes and half the gather instructions of the single-block kernel (K3 is bound
// by its gathers: profiles/r2_k3_split.txt).  The rest of each block's list (and the
// compensator rows) then runs in down_proj_kernel, which adds onto these Y tiles.
#include "ffwd_internal.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace ffwd {

namespace {

constexpr int PBM = 128;                // token rows per CTA (one block)
constexpr int PBK = 64;                 // K rows per stage
constexpr int PBN = 256;                // output columns of a pair tile
constexpr int kHalfN = PBN / 2;         // columns each CTA gathers
constexpr int kPStages = 7;
constexpr int kPA = PBM * PBK * 2;      // 16 KiB: the block's H tile
constexpr int kPB = PBK * kHalfN * 2;   // 16 KiB: this CTA's half of the gathered rows
constexpr int kPStage = kPA + kPB;
constexpr int kPProducers = 8;
constexpr int kPEpi0 = kPProducers;     // warps 8..11: epilogue (warp % 4 = TMEM lane quadrant)
constexpr int kPMma = kPProducers + 4;  // warp 12: TMEM allocator; the leader's MMA issuer
constexpr int kPThreads = (kPProducers + 5) * 32;
constexpr int kPQ = PBK / kPProducers;  // K rows per producer warp and stage
constexpr uint32_t kPLbo = (PBK / 8) * 1024;  // MN-major B: 64-column atom stride

struct PairBars {
  uint64_t full[kPStages];   // leader: both CTAs' A + B bytes of the stage landed
  uint64_t empty[kPStages];  // both CTAs: the pair's MMAs released the stage
  uint64_t tfull[2];
  uint64_t tempty[2];        // leader: both CTAs' epilogues drained the accumulator
  uint32_t tmem_base;
  uint32_t pad;
  alignas(16) int rows[kPProducers][kPQ];
};

constexpr size_t kPairSmem = 1024 + static_cast<size_t>(kPStages) * kPStage + sizeof(PairBars);

__device__ __forceinline__ void wait_done(const int* done, int n) {
  for (long long spins = 0;; ++spins) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    if (v >= n) break;
    __nanosleep(200);
    if (spins > (1ll << 26)) __trap();  // the up projection never published this block
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPThreads, 1)
    down_pair_kernel(const __grid_constant__ CUtensorMap tm_h,
                     const __grid_constant__ CUtensorMap tm_w, PairArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  PairBars* bar = reinterpret_cast<PairBars*>(base + kPStages * kPStage);
  auto a_st = [&](int s) { return base + s * kPStage; };
  auto b_st = [&](int s) { return base + s * kPStage + kPA; };
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int cl = static_cast<int>(blockIdx.x >> 1), ncl = static_cast<int>(gridDim.x >> 1);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_h);
    tma_prefetch_desc(&tm_w);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&bar->full[s], 1);
      mbar_init(&bar->empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar->tfull[i], 1);
      mbar_init(&bar->tempty[i], 2);
    }
    fence_barrier_init();
  }
  if (warp == kPMma) tmem_alloc_cg2<512>(&bar->tmem_base);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers and TMEM before any cross-CTA traffic
  tc_fence_after();
  if (!a.blk_done) pdl_wait();
  pdl_trigger();
  const uint32_t tmem = bar->tmem_base;
  const int n_tiles = a.n_tiles;

  if (warp < kPProducers) {
    // ---------------- producers: warp w gathers K rows [Q w, Q w + Q) of every stage, this
    // CTA's 128 columns; warp 0 also loads the block's H tile (and, in the leader, expects
    // the stage's bytes of both CTAs)
    const uint64_t pol_h = policy_evict_last(), pol_w = policy_evict_normal();
    int* rows = bar->rows[warp];
    uint32_t stage = 0, phase = 0;
    for (int t = cl; t < n_tiles; t += ncl) {
      const PairTile pt = a.tiles[t];
      if (pt.b0 < 0) continue;
      const int b = rank ? pt.b1 : pt.b0;
      const int32_t* list = a.idx + static_cast<size_t>(pt.row) * a.ld_idx;
      for (int kb = 0; kb < pt.nk; ++kb) {
        if (lane < static_cast<uint32_t>(kPQ)) rows[lane] = __ldg(list + kb * PBK + kPQ * warp + lane);
        __syncwarp();
        if (lane == 0) {
          mbar_wait(&bar->empty[stage], phase ^ 1);
          if (warp == 0) {
#ifndef FFWD_PAIR_EXPT
            if (rank == 0) mbar_arrive_expect_tx(&bar->full[stage], 2 * kPStage);
#elif FFWD_PAIR_EXPT == 1  // timing only: no B gathers
            if (rank == 0) mbar_arrive_expect_tx(&bar->full[stage], 2 * kPA);
#else                      // timing only: no A loads
            if (rank == 0) mbar_arrive_expect_tx(&bar->full[stage], 2 * kPB);
#endif
            if (kb == 0 && a.blk_done) wait_done(a.blk_done + b, a.meta[b].n_up);
#if !defined(FFWD_PAIR_EXPT) || FFWD_PAIR_EXPT != 2
            tma_load_2d_cg2(&tm_h, &bar->full[stage], a_st(stage), kb * PBK, b * PBM, pol_h);
#endif
          }
#if defined(FFWD_PAIR_EXPT) && FFWD_PAIR_EXPT == 1
          constexpr int kGatherQ = 0;
#else
          constexpr int kGatherQ = kPQ / 4;
#endif
          const int4* rq = reinterpret_cast<const int4*>(rows);
#pragma unroll
          for (int q = 0; q < kGatherQ; ++q) {
            const int4 r = rq[q];
            const int pos = kPQ * warp + 4 * q;  // K row within the stage
            uint8_t* dst = b_st(stage) + (pos >> 3) * 1024 + (pos & 7) * 128;
#pragma unroll
            for (int c = 0; c < kHalfN / 64; ++c)
              tma_gather4_cg2(&tm_w, &bar->full[stage], dst + c * kPLbo,
                              pt.n0 + static_cast<int>(rank) * kHalfN + c * 64, r.x, r.y, r.z,
                              r.w, pol_w);
          }
        }
        __syncwarp();
        if (++stage == kPStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == kPMma) {
    // ---------------- the leader's single MMA-issuing thread
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(2 * PBM, PBN, false, true);
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int t = cl; t < n_tiles; t += ncl) {
        const PairTile pt = a.tiles[t];
        if (pt.b0 < 0) continue;
        mbar_wait_sleep(&bar->tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < pt.nk; ++kb) {
          mbar_wait(&bar->full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = make_sdesc_sw128(smem_u32(a_st(stage)), 16, 1024);
          const uint64_t bdesc = make_sdesc_sw128(smem_u32(b_st(stage)), kPLbo, 1024);
#pragma unroll
          for (int kk = 0; kk < PBK / 16; ++kk)
            umma_bf16_cg2(tmem + acc * PBN, adesc + static_cast<uint64_t>(2 * kk),
                          bdesc + static_cast<uint64_t>((2048 >> 4) * kk), idesc,
                          (kb | kk) != 0 ? 1u : 0u);
          umma_commit_cg2_mc(&bar->empty[stage], 0x3);
          if (++stage == kPStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_cg2_mc(&bar->tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (both CTAs): this CTA's block rows of the pair tile
    const int ew = warp - kPEpi0;
    const int row = ew * 32 + static_cast<int>(lane);
    uint32_t acc = 0, acc_phase = 0;
    for (int t = cl; t < n_tiles; t += ncl) {
      const PairTile pt = a.tiles[t];
      if (pt.b0 < 0) continue;
      const int b = rank ? pt.b1 : pt.b0;
      mbar_wait_sleep(&bar->tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem + acc * PBN + (static_cast<uint32_t>(ew * 32) << 16);
      const int ntok = min(PBM, a.T - b * PBM);
      const size_t row_off = static_cast<size_t>(b * PBM + row) * a.d + pt.n0;
#pragma unroll 1
      for (int c = 0; c < PBN; c += 16) {
        uint32_t v[16];
        tmem_ld16(tb + c, v);
        tmem_ld_wait();
        if (row < ntok) {
          float o[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = __uint_as_float(v[j]);
          if (a.residual) {
            const float4* res = reinterpret_cast<const float4*>(a.residual + row_off + c);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 r = res[j];
              o[4 * j] += r.x;
              o[4 * j + 1] += r.y;
              o[4 * j + 2] += r.z;
              o[4 * j + 3] += r.w;
            }
          }
          float4* dst = reinterpret_cast<float4*>(a.y + row_off + c);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        }
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (row == 0) mbar_arrive_cluster(&bar->tempty[acc], 0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA frees TMEM or leaves while its peer may still signal it
  tc_fence_after();
  if (warp == kPMma) tmem_dealloc_cg2<512>(tmem);
}

}  // namespace

cudaError_t launch_down_pair(const PairArgs& a, cudaStream_t s) {
  if (a.n_tiles <= 0) return cudaSuccess;
  if (a.d % PBN != 0) return cudaErrorInvalidValue;
  CUtensorMap th, tw;
  if (encode_tmap_2d_bf16(&th, a.h, a.hcols, static_cast<uint64_t>(a.n_blk) * PBM, PBK, PBM) !=
      CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&tw, a.wd, a.d, a.wd_rows, 64, 1) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = ensure_smem_limit(down_pair_kernel, kPairSmem, attr); e != cudaSuccess)
    return e;
  int grid = a.num_sms & ~1;
  const int need = 2 * a.n_tiles;
  if (grid > need) grid = need;
  if (grid < 2) grid = 2;
  return launch_k(down_pair_kernel, dim3(grid), dim3(kPThreads), kPairSmem, s, 1, th, tw, a);
}

}  // namespace ffwd

#ifdef FFWD_PAIR_BENCH
// Timing / correctness harness (build variant only): pair i = blocks (2i, 2i+1), both using
// index row 2i's first 64 nk entries; all d / 256 column tiles.
#include <vector>
extern "C" __attribute__((visibility("default"))) int ffwd_down_pair_bench(
    const void* h, int hcols, const void* wd, int wd_rows, int T, int d, float* y,
    const float* residual, const int32_t* idx, int ld_idx, int n_pairs, int nk, void* stream) {
  using namespace ffwd;
  static PairTile* dev_tiles = nullptr;
  static int cap = 0;
  const int nt = d / 256;
  std::vector<PairTile> t;  // raster: groups of 8 pairs, column-tile major inside a group
  for (int g0 = 0; g0 < n_pairs; g0 += 8)
    for (int j = 0; j < nt; ++j)
      for (int i = g0; i < n_pairs && i < g0 + 8; ++i)
        t.push_back(PairTile{2 * i, 2 * i + 1, j * 256, nk, 2 * i, 0, 0, 0});
  if (static_cast<int>(t.size()) > cap) {
    if (dev_tiles) cudaFree(dev_tiles);
    cap = static_cast<int>(t.size());
    if (cudaMalloc(&dev_tiles, cap * sizeof(PairTile)) != cudaSuccess) return 2;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemcpyAsync(dev_tiles, t.data(), t.size() * sizeof(PairTile), cudaMemcpyHostToDevice, s);
  PairArgs a{};
  a.h = h;
  a.hcols = hcols;
  a.wd = wd;
  a.wd_rows = wd_rows;
  a.T = T;
  a.d = d;
  a.n_blk = (T + 127) / 128;
  a.y = y;
  a.residual = residual;
  a.idx = idx;
  a.ld_idx = ld_idx;
  a.tiles = dev_tiles;
  a.n_tiles = static_cast<int>(t.size());
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  a.num_sms = sms;
  return launch_down_pair(a, s) == cudaSuccess ? 0 : 2;
}
#endif
