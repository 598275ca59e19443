// K2: up projection of the sparse SwiGLU FFN as a tcgen05 gather-GEMM.
//
//   H_b[:, p] = silu(X_b . Wg[:, idx_b[p]]) * (X_b . Wu[:, idx_b[p]])   p < k_b
//   (sparse.py:81-91: gate / up matmuls + kernels.silu, for one 128-token block b)
//   C_b       = silu(X_b . Wc1)                                            comp tiles
//   (compensator.py:52-58 hidden layer, predicted blocks only, engine.py:296)
//
// A = X_b (128 x 64 per stage) by 2-D TMA; B = the selected rows of the
// neuron-major [gate^T | up^T | Wc1^T] (bf16, K-major) by TMA tile::gather4,
// 128 gate + 128 up rows per gate/up tile (or 256 Wc1 rows per comp tile);
// D = 128 x 256 f32 in TMEM; SiLU(gate) * up fused in the TMEM -> register
// epilogue, written as bf16 into H (row stride hcols, block b at rows 128 b).
// 16 issuing warps: gathers here are 128 B rows at 8 KiB stride, the up projection is
// gather-rate bound (r1 A/B: 2.39 -> 2.21 ms/layer vs 8 warps).
#ifndef FFWD_UP_PRODUCERS
#define FFWD_UP_PRODUCERS 16
#endif
#define FFWD_PRODUCER_WARPS FFWD_UP_PRODUCERS
// B (the gathers) gets a 5-deep ring and A a 4-deep one loaded by its own warp (smem
// 4 x 16 + 5 x 32 KiB); the two CTAs of a cluster run neuron tiles (i, i+1) of the same
// token block and each loads half of the block's X tile, multicast to both.
#ifndef FFWD_UP_UNSPLIT
#define FFWD_SPLIT_RING
// CTA pairs sharing X by TMA multicast (L2->SM bytes -11%, in-stack K2 -1.5..2.7%).
#ifndef FFWD_UP_NOPAIR
#define FFWD_PAIR_A
#endif
#ifndef FFWD_STAGES_A
#define FFWD_STAGES_A 4
#endif
#ifndef FFWD_STAGES_B
#define FFWD_STAGES_B 5
#endif
#endif
// Dynamic tile claiming (FFWD_K2_DYN, default on; CTA pairs claim slot pairs together)
#ifndef FFWD_K2_DYN
#define FFWD_K2_DYN 1
#endif
#if FFWD_K2_DYN
#define FFWD_DYN_TILES
#endif
#include "gemm_sm100.cuh"
#include "launch.cuh"

// L2 prefetch distance of the gathered gate/up rows, in K stages (0 = off, measured slower
// at 4/8/16: profiles/r2_prefetch_ab.txt; a multiple of
// 4): every 4 stages each producer warp prefetches its rows' next 4 column chunks
// (256 columns, tile::gather4 prefetch) P stages ahead of the gathers.
#ifndef FFWD_K2_PREFETCH
#define FFWD_K2_PREFETCH 0
#endif

namespace ffwd {

namespace {
#ifdef FFWD_PROBE
__device__ unsigned long long g_probe_up[256][5];  // per CTA: wait A, wait B, wait TMEM, total, stages
#endif

using namespace gemm;

constexpr int UP_BN = 256;
constexpr int kBBytes = UP_BN * BK * 2;  // 32 KiB per stage

__global__ void __launch_bounds__(kThreads, 1)
    up_proj_kernel(const __grid_constant__ CUtensorMap tm_x,
                   const __grid_constant__ CUtensorMap tm_w,
                   const __grid_constant__ CUtensorMap tm_wt,
                   const __grid_constant__ CUtensorMap tm_xh,
                   const __grid_constant__ CUtensorMap tm_wpf, GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  Smem<kBBytes> sm(smem_raw);
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_wt);
  }
  prologue(sm, warp);
  pdl_wait();  // the prologue overlapped the predecessor; tile tables, X, idx are its output
  pdl_trigger();
  const uint32_t tmem = sm.bar->tmem_base;
  const int n_tiles = a.counts->n_up;
  // every role walks the same tile sequence: claimed dynamically by producer warp 0 (of
  // rank 0 for a CTA pair) or strided
  TileCursor cur;
  int* const claim_ctr = &a.counts->next_up;
  const uint32_t crank = kPairA ? cluster_ctarank() : 0;
  auto fetch = [&](bool warp_wide) -> int {
    if constexpr (kPairA) {
      return (warp == 0 && crank == 0) ? cur.claim_pair(&sm.bar->q, claim_ctr, n_tiles)
                                       : cur.next_pair(&sm.bar->q, warp_wide, crank);
    } else {
      return warp == 0 ? cur.claim(&sm.bar->q, claim_ctr, n_tiles)
                       : cur.next(&sm.bar->q, warp_wide);
    }
  };
  auto first_tile = [&](bool warp_wide) {
    return kDyn ? fetch(warp_wide) : static_cast<int>(blockIdx.x);
  };
  auto next_tile = [&](int t, bool warp_wide) {
    return kDyn ? fetch(warp_wide) : t + static_cast<int>(gridDim.x);
  };
  auto more = [&](int t) { return kDyn ? t >= 0 : t < n_tiles; };
  const int nk = a.d / BK;

  if (warp < kProducerWarps) {
    // ---------------- producers: warp w gathers B rows [R w, R w + R) of every stage
    constexpr int R = UP_BN / kProducerWarps;  // rows per producer warp
#ifndef FFWD_K2_W_POLICY
#define FFWD_K2_W_POLICY 0
#endif
    const uint64_t pol_x = policy_evict_last();
    const uint64_t pol_w = FFWD_K2_W_POLICY == 2 ? policy_evict_last()
                           : FFWD_K2_W_POLICY == 1 ? policy_evict_first() : policy_evict_normal();
    int* rows = sm.bar->rows[warp];
    uint32_t stage = 0, phase = 0;
    for (int t = first_tile(true); more(t); t = next_tile(t, true)) {
      const Tile tl = a.up_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      // Contiguous B rows (dense blocks' identity index, compensator rows) take the
      // 2-D tile path: two 128-row boxes issued by warp 0, ~1.5x the gather4 rate.
      const bool contiguous = tl.kind != 0 || m.idx_row < 0;
      if (!contiguous) {
        for (int i = static_cast<int>(lane); i < R; i += 32) {
          const int j = R * warp + i;  // B row within the tile
          const int half = j >> 7;     // 0 = gate rows, 1 = up rows
          rows[i] = neuron_at(m, a.idx, a.ld_idx, tl.n0 + (j & 127)) + half * a.f_local;
        }
      }
      __syncwarp();
      if (lane == 0) {
        uint32_t bytes = contiguous ? 0 : R * BK * 2;
        if (warp == 0) bytes += (kSplit ? 0 : kABytes) + (contiguous ? UP_BN * BK * 2 : 0);
        const int r0 = tl.kind != 0 ? 2 * a.f_local + tl.n0 : tl.n0;  // first box row
        const int r1 = tl.kind != 0 ? r0 + 128 : a.f_local + tl.n0;    // second box row
        const int4* rq = reinterpret_cast<const int4*>(rows);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&sm.bar->empty[stage], phase ^ 1);
          if (bytes)
            mbar_arrive_expect_tx(&sm.bar->full[stage], bytes);
          else
            mbar_arrive(&sm.bar->full[stage]);
          if (warp == 0) {
            if (!kSplit)
              tma_load_2d(&tm_x, &sm.bar->full[stage], sm.a_stage(stage), kb * BK, m.tok0,
                          pol_x);
            if (contiguous) {
              tma_load_2d(&tm_wt, &sm.bar->full[stage], sm.b_stage(stage), kb * BK, r0, pol_w);
              tma_load_2d(&tm_wt, &sm.bar->full[stage], sm.b_stage(stage) + 128 * 128, kb * BK,
                          r1, pol_w);
            }
          }
          if constexpr (FFWD_K2_PREFETCH > 0) {
            const int kp = kb + FFWD_K2_PREFETCH;
            if (!contiguous && (kb & 3) == 0 && kp < nk) {
#pragma unroll
              for (int q = 0; q < R / 4; ++q) {
                const int4 r = rq[q];
                tma_prefetch_gather4(&tm_wpf, kp * BK, r.x, r.y, r.z, r.w);
              }
            }
          }
          if (!contiguous) {
            uint8_t* dst = sm.b_stage(stage) + warp * R * 128;
#pragma unroll
            for (int q = 0; q < R / 4; ++q) {
              const int4 r = rq[q];
              tma_gather4(&tm_w, &sm.bar->full[stage], dst + q * 512, kb * BK, r.x, r.y, r.z,
                          r.w, pol_w);
            }
          }
          advance(stage, phase);
        }
      }
      __syncwarp();
    }
  } else if (kSplit && warp == kAWarp) {
    // ---------------- A loader (split rings): the block's X tile, one 2-D box per stage
    if (lane == 0) {
#ifndef FFWD_K2_X_POLICY
#define FFWD_K2_X_POLICY 2
#endif
      const uint64_t pol_x = FFWD_K2_X_POLICY == 2 ? policy_evict_last()
                             : FFWD_K2_X_POLICY == 1 ? policy_evict_first() : policy_evict_normal();
      uint32_t sa = 0, pa = 0;
      for (int t = first_tile(false); more(t); t = next_tile(t, false)) {
        const Tile tl = a.up_tiles[t];
        if (tl.b < 0) continue;
        const int tok0 = a.meta[tl.b].tok0;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&sm.bar->emptyA[sa], pa ^ 1);  // paired: both CTAs' MMAs released it
          mbar_arrive_expect_tx(&sm.bar->fullA[sa], kABytes);
          if constexpr (kPairA) {  // my 64-row half of X_b, multicast to both CTAs
            const uint32_t cr = cluster_ctarank();
            tma_load_2d_mc(&tm_xh, &sm.bar->fullA[sa], sm.a_stage(sa) + cr * (kABytes / 2),
                           kb * BK, tok0 + static_cast<int>(cr) * (BM / 2), 0x3, pol_x);
          } else {
            tma_load_2d(&tm_x, &sm.bar->fullA[sa], sm.a_stage(sa), kb * BK, tok0, pol_x);
          }
          advance_n<kStagesA>(sa, pa);
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = make_idesc_bf16(BM, UP_BN, false, false);
    if (lane == 0) {
      Probe pr;
#ifdef FFWD_PROBE
      pr.t0 = clock64();
#endif
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0, sa = 0, pa = 0;
      for (int t = first_tile(false); more(t); t = next_tile(t, false)) {
        const Tile tl = a.up_tiles[t];
        if (tl.b < 0) continue;
#ifdef FFWD_PROBE
        const unsigned long long ct = clock64();
        mbar_wait_sleep(&sm.bar->tempty[acc], acc_phase ^ 1);
        pr.wait_t += clock64() - ct;
#else
        mbar_wait_sleep(&sm.bar->tempty[acc], acc_phase ^ 1);
#endif
        tc_fence_after();
        if constexpr (kSplit)
          mma_tile_split(sm, tmem + acc * UP_BN, nk, idesc, 16, 1024, 32, stage, phase, sa, pa, &pr);
        else
          mma_tile(sm, tmem + acc * UP_BN, nk, idesc, 16, 1024, 32, stage, phase);
        umma_commit(&sm.bar->tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
#ifdef FFWD_PROBE
      if (blockIdx.x < 256) {
        unsigned long long* o = g_probe_up[blockIdx.x];
        o[0] = pr.wait_a; o[1] = pr.wait_b; o[2] = pr.wait_t; o[3] = clock64() - pr.t0;
        o[4] = pr.stages;
      }
#endif
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: TMEM -> regs -> SiLU(g) * u -> bf16 H
    const int ew = warp - kEpiWarp0;
    const int row = ew * 32 + static_cast<int>(lane);
    uint32_t acc = 0, acc_phase = 0;
    for (int t = first_tile(true); more(t); t = next_tile(t, true)) {
      const Tile tl = a.up_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      mbar_wait_sleep(&sm.bar->tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem + acc * UP_BN + (static_cast<uint32_t>(ew * 32) << 16);
      __nv_bfloat16* hrow = static_cast<__nv_bfloat16*>(a.h) +
                            static_cast<size_t>(tl.b * kBlockTokens + row) * a.hcols;
      // 16-column chunks keep the epilogue's register footprint small enough for
      // 16 producer warps in the same CTA.
      if (tl.kind == 0) {
#pragma unroll 1
        for (int c = 0; c < 128; c += 16) {
          const int pos = tl.n0 + c;
          if (pos >= m.kpad) break;
          uint32_t g[16], u[16];
          tmem_ld16(tb + c, g);
          tmem_ld16(tb + 128 + c, u);
          tmem_ld_wait();
          uint32_t packed[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float h0 = silu_f32(__uint_as_float(g[2 * j])) * __uint_as_float(u[2 * j]);
            float h1 = silu_f32(__uint_as_float(g[2 * j + 1])) * __uint_as_float(u[2 * j + 1]);
            if (pos + 2 * j >= m.kcount) h0 = 0.0f;
            if (pos + 2 * j + 1 >= m.kcount) h1 = 0.0f;
            packed[j] = pack_bf16x2(h0, h1);
          }
          uint4* dst = reinterpret_cast<uint4*>(hrow + pos);
          dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < UP_BN; c += 16) {
          const int col = tl.n0 + c;
          if (col >= m.comp) break;
          uint32_t g[16];
          tmem_ld16(tb + c, g);
          tmem_ld_wait();
          uint32_t packed[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            packed[j] = pack_bf16x2(silu_f32(__uint_as_float(g[2 * j])),
                                    silu_f32(__uint_as_float(g[2 * j + 1])));
          uint4* dst = reinterpret_cast<uint4*>(hrow + m.kpad + col);
          dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        }
      }
      if (a.blk_done) {  // publish "one more H tile of block b is written" (K3 waits on it)
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (row == 0) atomicAdd(a.blk_done + tl.b, 1);
      }
      tc_fence_before();
      mbar_arrive(&sm.bar->tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  teardown(sm, warp);
}

}  // namespace

bool up_proj_paired() { return kPairA; }

cudaError_t launch_up_proj(const GemmArgs& a, cudaStream_t s) {
  CUtensorMap tx, tw, twt, txh;
  if (encode_tmap_2d_bf16(&tx, a.x, a.d, a.T, BK, BM) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&txh, a.x, a.d, a.T, BK, BM / 2) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&tw, a.wgu_t, a.d, a.wgu_rows, BK, 1) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&twt, a.wgu_t, a.d, a.wgu_rows, BK, 128) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  CUtensorMap twpf;  // L2 prefetch: 4 column chunks of 4 gathered rows per instruction
  if (encode_tmap_2d_bf16_sw(&twpf, a.wgu_t, a.d, a.wgu_rows, 4 * BK, 1, false) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  constexpr size_t smem = smem_bytes<kBBytes>();
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = ensure_smem_limit(up_proj_kernel, smem, attr); e != cudaSuccess) return e;
  int grid = a.num_sms < a.up_cap ? a.num_sms : a.up_cap;
  if constexpr (kPairA) {
    grid &= ~1;  // whole CTA pairs; the plan pads the tile table to pairs
    if (grid < 2) grid = 2;
  }
  return launch_k(up_proj_kernel, dim3(grid), dim3(kThreads), smem, s, kPairA ? 2 : 1, tx, tw, twt,
                  txh, twpf, a);
}

}  // namespace ffwd

#ifdef FFWD_PROBE
extern "C" __attribute__((visibility("default"))) int ffwd_probe_read_up(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, ffwd::g_probe_up, sizeof(ffwd::g_probe_up)) == cudaSuccess ? 0 : 1;
}
#endif
