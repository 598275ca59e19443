// K3: down projection + low-rank compensator as one tcgen05 gather-GEMM.
//
//   Y_b = [H_b | C_b] . [W_down[idx_b, :] ; Wc2]
//   (sparse.py:91 down matmul + compensator.py:52-66: silu(x Wc1) Wc2 added to
//   the output -- here simply r' extra K iterations into the same TMEM
//   accumulator, so the correction is fused into the down-projection accumulate)
//
// A = H_b (128 x 64 per stage, K-major) by 2-D TMA; B = the stage's 64 K rows
// (selected neurons, then compensator rows) of [W_down ; Wc2] (bf16, d
// contiguous = MN-major) by TMA tile::gather4 in BN/64 column atoms; D = 128 x BN
// f32 in TMEM.  Epilogue: optional residual add (engine.py:308) and optional
// bf16 copy for the next layer's input, f32 Y stores.
// 8 issuing warps (r1 A/B: 16 warps gave no gain here: 1.07 vs 1.09 ms/layer).
#ifndef FFWD_DOWN_PRODUCERS
#define FFWD_DOWN_PRODUCERS 8
#endif
#define FFWD_PRODUCER_WARPS FFWD_DOWN_PRODUCERS
#define FFWD_GATHER_ROWS 64  // BK K rows per stage
// Split rings as in K2 (A = H on its own loader warp, 4-deep; gathered B 5-deep; 224 KiB):
// on by default (FFWD_DOWN_UNSPLIT: one shared ring, A loaded by producer warp 0).  r1 A/B,
// two boxes: K3 2-5% faster in the stack (1.12 -> 1.06 and 1.17 -> 1.11 ms/layer), tensor
// pipe 55.9 -> 59.4% under ncu.
// Option (off): CTA pairs (FFWD_DOWN_PAIR: the two CTAs of a cluster run column tiles
// (j, j+1) of one block and each loads half of its H tile, multicast to both).  ncu,
// 8B/16K: pairs cut K3's L2->SM bytes 6.8% but raise its DRAM reads from 1.64 to 2.0-2.4 GB
// for every raster group size, and are within noise in the stack.
#ifdef FFWD_DOWN_PAIR
#define FFWD_PAIR_A
#endif
#if !defined(FFWD_DOWN_UNSPLIT) || defined(FFWD_DOWN_PAIR)
#define FFWD_SPLIT_RING
#ifndef FFWD_DOWN_STAGES_A
#define FFWD_DOWN_STAGES_A 4
#endif
#ifndef FFWD_DOWN_STAGES_B
#define FFWD_DOWN_STAGES_B 5
#endif
#define FFWD_STAGES_A FFWD_DOWN_STAGES_A
#define FFWD_STAGES_B FFWD_DOWN_STAGES_B
#endif
// FFWD_K3_A_LDGSTS: H tiles by cp.async from the A-loader warp instead of TMA boxes
#ifdef FFWD_K3_A_LDGSTS
#define FFWD_A_LDGSTS
#endif
// FFWD_K3_B_LDGSTS: the gathered W_down rows by 16 B cp.async from all producer lanes
// instead of TMA tile::gather4 (contiguous stages keep their 2-D TMA boxes)
#ifdef FFWD_K3_B_LDGSTS
#define FFWD_B_LDGSTS
#endif
// Dynamic tile claiming (FFWD_K3_DYN, default on): gemm_sm100.cuh TileQueue.
#ifndef FFWD_K3_DYN
#define FFWD_K3_DYN 1
#endif
#if FFWD_K3_DYN
#define FFWD_DYN_TILES
#endif
#include "gemm_sm100.cuh"
#include "launch.cuh"

// L2 policies (A/B tuning knobs): 0 evict_normal, 1 evict_first, 2 evict_last.
#ifndef FFWD_K3_H_POLICY
#define FFWD_K3_H_POLICY 2
#endif
#ifndef FFWD_K3_W_POLICY
#define FFWD_K3_W_POLICY 0
#endif
// L2 prefetch distance of the gathered W_down rows, in K stages (0 = off; measured slower
// at 2/4/8: profiles/r2_prefetch_ab.txt): each producer
// warp prefetches its rows of stage kb + P (tile::gather4 prefetch, one instruction per 4
// rows x BN columns) while it gathers stage kb.
#ifndef FFWD_K3_PREFETCH
#define FFWD_K3_PREFETCH 0
#endif
// 1: residual loads / Y and next-X stores bypass L2 residency (.cs streaming)
#ifndef FFWD_K3_STREAM_EPI
#define FFWD_K3_STREAM_EPI 0
#endif

namespace ffwd {

namespace {
#ifdef FFWD_PROBE
__device__ unsigned long long g_probe_down[256][5];  // per CTA: wait A, wait B, wait TMEM, total, stages
#endif

using namespace gemm;

// Spin until all `n` up-projection tiles of a block have published their H (K2 epilogue
// counters), then make the writes visible to this thread's TMA loads.  Bounded: traps
// after ~10 s rather than hanging the GPU.
__device__ __forceinline__ void wait_block_h(const int* done, int n) {
  for (long long spins = 0;; ++spins) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    if (v >= n) break;
    __nanosleep(200);
    if (spins > (1ll << 26)) __trap();  // K2 never published this block: fail, do not hang
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    down_proj_kernel(const __grid_constant__ CUtensorMap tm_h,
                     const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ CUtensorMap tm_wt,
                     const __grid_constant__ CUtensorMap tm_hh,
                     const __grid_constant__ CUtensorMap tm_wpf, GemmArgs a) {
  constexpr int kBBytes = BK * BN * 2;
  constexpr int kChunks = BN / 64;            // 64-column (128 B) atoms along N
  constexpr uint32_t kLbo = (BK / 8) * 1024;  // MN-direction atom stride
  extern __shared__ uint8_t smem_raw[];
  Smem<kBBytes> sm(smem_raw);
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_h);
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_wt);
  }
  prologue(sm, warp);
  // The tile tables come from the plan, which K2 waited for before letting K3 launch.
  // With per-block counters K3 waits only for the H of the block each tile reads (A
  // loads below), so its first tiles overlap K2's tail; otherwise wait for all of K2.
  if (!a.blk_done) pdl_wait();
  pdl_trigger();
  const uint32_t tmem = sm.bar->tmem_base;
  const int n_tiles = a.counts->n_down;
  // every role walks the same tile sequence: claimed dynamically (TileQueue) or strided
  // (producer warp 0 claims; the other roles follow its sequence)
  TileCursor cur;
  int* const claim_ctr = &a.counts->next_down;
  auto fetch = [&](bool warp_wide) {
    return warp == 0 ? cur.claim(&sm.bar->q, claim_ctr, n_tiles) : cur.next(&sm.bar->q, warp_wide);
  };
  auto first_tile = [&](bool warp_wide) {
    return kDyn ? fetch(warp_wide) : static_cast<int>(blockIdx.x);
  };
  auto next_tile = [&](int t, bool warp_wide) {
    return kDyn ? fetch(warp_wide) : t + static_cast<int>(gridDim.x);
  };
  auto more = [&](int t) { return kDyn ? t >= 0 : t < n_tiles; };

  if (warp < kProducerWarps) {
    // ---------------- producers: warp w gathers K rows [Q w, Q w + Q) of every stage
    constexpr int Q = BK / kProducerWarps;  // K rows per producer warp (multiple of 4)
    auto pol = [](int k) {
      return k == 1 ? policy_evict_first() : (k == 2 ? policy_evict_last() : policy_evict_normal());
    };
    const uint64_t pol_h = pol(FFWD_K3_H_POLICY);
    const uint64_t pol_w = pol(FFWD_K3_W_POLICY);
    int* rows = sm.bar->rows[warp];
    uint32_t stage = 0, phase = 0;
    for (int t = first_tile(true); more(t); t = next_tile(t, true)) {
      const Tile tl = a.down_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      const int nk = m.ktot / BK;
      // Tile.pad = 1: this tile walks its K stages from the top down (serpentine raster:
      // the W_down rows the previous group read last are still in L2)
      auto kidx = [&](int kb) { return tl.pad ? nk - 1 - kb : kb; };
      auto row_of = [&](int kb) -> int {
        const int p = kidx(kb) * BK + Q * warp + static_cast<int>(lane % Q);
        return p < m.kpad ? neuron_at(m, a.idx, a.ld_idx, p) : a.f_local + (p - m.kpad);
      };
      // Neuron ids are prefetched 4 stages ahead (a register ring): an index load that
      // misses L2 outlasts one stage, and the gathers of a stage cannot issue without it.
      int r0 = row_of(0), r1 = nk > 1 ? row_of(1) : 0, r2 = nk > 2 ? row_of(2) : 0,
          r3 = nk > 3 ? row_of(3) : 0;
      for (int kb = 0; kb < nk; ++kb) {
        const int cur = r0;
        r0 = r1;
        r1 = r2;
        r2 = r3;
        if (kb + 4 < nk) r3 = row_of(kb + 4);
        // Contiguous K rows (identity index of dense blocks, compensator rows past kpad)
        // take the 2-D tile path: one 64-row box per column atom, issued by warp 0.
        const int kr = kidx(kb);  // K stage actually loaded (reversed tiles sweep downwards)
        const bool contiguous = m.idx_row < 0 || kr * BK >= m.kpad;
        if constexpr (FFWD_K3_PREFETCH > 0) {
          // warm L2 with this warp's rows of stage kb + P (gathered P stages from now)
          const int kp = kb + FFWD_K3_PREFETCH;
          const bool pf = kp < nk && m.idx_row >= 0 && kidx(kp) * BK < m.kpad;
          const int prow = pf ? row_of(kp) : 0;
#pragma unroll
          for (int q = 0; q < Q / 4; ++q) {
            const int p0 = __shfl_sync(0xffffffffu, prow, 4 * q);
            const int p1 = __shfl_sync(0xffffffffu, prow, 4 * q + 1);
            const int p2 = __shfl_sync(0xffffffffu, prow, 4 * q + 2);
            const int p3 = __shfl_sync(0xffffffffu, prow, 4 * q + 3);
            if (pf && lane == 0) tma_prefetch_gather4(&tm_wpf, tl.n0, p0, p1, p2, p3);
          }
        }
        if (lane < Q) rows[lane] = cur;
        __syncwarp();
        if constexpr (kBLdgsts) {
          static_assert(kSplit, "B by cp.async needs the split A ring");
          if (lane == 0) mbar_wait(&sm.bar->empty[stage], phase ^ 1);
          __syncwarp();
          if (contiguous) {
            if (warp == 0 && lane == 0) {
              mbar_arrive_expect_tx(&sm.bar->full[stage], BK * BN * 2);
              if (kb == 0 && a.blk_done) wait_block_h(a.blk_done + tl.b, m.n_up);
              const int r0 = m.idx_row < 0 ? kr * BK : a.f_local + (kr * BK - m.kpad);
#pragma unroll
              for (int c = 0; c < kChunks; ++c)
                tma_load_2d(&tm_wt, &sm.bar->full[stage], sm.b_stage(stage) + c * kLbo,
                            tl.n0 + c * 64, r0, pol_w);
            } else {
              mbar_arrive(&sm.bar->full[stage]);
            }
          } else {
            // lane l copies 16 B chunks l, l+32, ... of the warp's Q row segments (BN = 256:
            // one whole row per warp instruction, coalesced), into the swizzled MN-major
            // atoms: chunk j of column atom c of K row pos at c*LBO + (pos/8)*1024 +
            // (pos%8)*128 + ((j ^ pos%8) * 16), where the tensor map's 128B swizzle puts it
            constexpr int kRowChunks = BN / 8;
            const __nv_bfloat16* wd = static_cast<const __nv_bfloat16*>(a.wd);
#pragma unroll
            for (int q = static_cast<int>(lane); q < Q * kRowChunks; q += 32) {
              const int i = q / kRowChunks, cc = q % kRowChunks, c = cc >> 3, j = cc & 7;
              const int pos = Q * warp + i;
              uint8_t* dst = sm.b_stage(stage) + c * kLbo + (pos >> 3) * 1024 +
                             (pos & 7) * 128 + ((j ^ (pos & 7)) << 4);
              cp_async_cg16(dst, wd + static_cast<size_t>(rows[i]) * a.d + tl.n0 + c * 64 +
                                     j * 8);
            }
            cp_async_arrive_noinc(&sm.bar->full[stage]);
          }
        } else if (lane == 0) {
          mbar_wait(&sm.bar->empty[stage], phase ^ 1);
          uint32_t nbytes = contiguous ? 0 : Q * BN * 2;
          if (warp == 0) nbytes += (kSplit ? 0 : kABytes) + (contiguous ? BK * BN * 2 : 0);
          if (nbytes)
            mbar_arrive_expect_tx(&sm.bar->full[stage], nbytes);
          else
            mbar_arrive(&sm.bar->full[stage]);
          if (warp == 0) {
            if (kb == 0 && a.blk_done) wait_block_h(a.blk_done + tl.b, m.n_up);
            if (!kSplit)
              tma_load_2d(&tm_h, &sm.bar->full[stage], sm.a_stage(stage), kr * BK,
                          tl.b * kBlockTokens, pol_h);
            if (contiguous) {
              const int r0 = m.idx_row < 0 ? kr * BK : a.f_local + (kr * BK - m.kpad);
#pragma unroll
              for (int c = 0; c < kChunks; ++c)
                tma_load_2d(&tm_wt, &sm.bar->full[stage], sm.b_stage(stage) + c * kLbo,
                            tl.n0 + c * 64, r0, pol_w);
            }
          }
          if (!contiguous) {
            const int4* rq = reinterpret_cast<const int4*>(rows);
#pragma unroll
            for (int q = 0; q < Q / 4; ++q) {
              const int4 r = rq[q];
              const int pos = Q * warp + 4 * q;  // K row within the stage
              uint8_t* dst = sm.b_stage(stage) + (pos >> 3) * 1024 + (pos & 7) * 128;
#pragma unroll
              for (int c = 0; c < kChunks; ++c)
                tma_gather4(&tm_w, &sm.bar->full[stage], dst + c * kLbo, tl.n0 + c * 64, r.x,
                            r.y, r.z, r.w, pol_w);
            }
          }
        }
        __syncwarp();
        advance(stage, phase);
      }
    }
  } else if (kSplit && kALdgsts && warp == kAWarp) {
    // ---------------- A loader, LSU path: the block's H tile by 16 B cp.async, written in
    // the 128B-swizzled K-major layout the UMMA descriptor expects (16 B chunk c of row r
    // at r * 128 + ((c ^ (r & 7)) * 16))
    uint32_t sa = 0, pa = 0;
    const __nv_bfloat16* H = static_cast<const __nv_bfloat16*>(a.h);
    for (int t = first_tile(true); more(t); t = next_tile(t, true)) {
      const Tile tl = a.down_tiles[t];
      if (tl.b < 0) continue;
      const int nk = a.meta[tl.b].ktot / BK;
      if (a.blk_done) {
        if (lane == 0) wait_block_h(a.blk_done + tl.b, a.meta[tl.b].n_up);
        __syncwarp();
      }
      const __nv_bfloat16* hb = H + static_cast<size_t>(tl.b) * kBlockTokens * a.hcols;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&sm.bar->emptyA[sa], pa ^ 1);
        const int kr = tl.pad ? nk - 1 - kb : kb;
        uint8_t* dst = sm.a_stage(sa);
#pragma unroll 8
        for (int i = 0; i < (BM * 8) / 32; ++i) {
          const int q = static_cast<int>(lane) + 32 * i;  // 16 B chunk of the tile
          const int r = q >> 3, c = q & 7;
          cp_async_cg16(dst + r * 128 + ((c ^ (r & 7)) << 4),
                        hb + static_cast<size_t>(r) * a.hcols + kr * BK + c * 8);
        }
        cp_async_arrive_noinc(&sm.bar->fullA[sa]);
        advance_n<kStagesA>(sa, pa);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
  } else if (kSplit && warp == kAWarp) {
    // ---------------- A loader (split rings): the block's H tile, one 2-D box per stage
    if (lane == 0) {
      const uint64_t pol_h = FFWD_K3_H_POLICY == 2 ? policy_evict_last()
                                                   : policy_evict_normal();
      uint32_t sa = 0, pa = 0;
      for (int t = first_tile(false); more(t); t = next_tile(t, false)) {
        const Tile tl = a.down_tiles[t];
        if (tl.b < 0) continue;
        const int nk = a.meta[tl.b].ktot / BK;
        if (a.blk_done) wait_block_h(a.blk_done + tl.b, a.meta[tl.b].n_up);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&sm.bar->emptyA[sa], pa ^ 1);
          mbar_arrive_expect_tx(&sm.bar->fullA[sa], kABytes);
          const int kr = tl.pad ? nk - 1 - kb : kb;
          if constexpr (kPairA) {  // my 64-row half of H_b, multicast to both CTAs
            const uint32_t cr = cluster_ctarank();
            tma_load_2d_mc(&tm_hh, &sm.bar->fullA[sa], sm.a_stage(sa) + cr * (kABytes / 2),
                           kr * BK, tl.b * kBlockTokens + static_cast<int>(cr) * (BM / 2), 0x3,
                           pol_h);
          } else {
            tma_load_2d(&tm_h, &sm.bar->fullA[sa], sm.a_stage(sa), kr * BK, tl.b * kBlockTokens,
                        pol_h);
          }
          advance_n<kStagesA>(sa, pa);
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    constexpr uint32_t idesc = make_idesc_bf16(BM, BN, false, true);
    if (lane == 0) {
      Probe pr;
#ifdef FFWD_PROBE
      pr.t0 = clock64();
#endif
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      [[maybe_unused]] uint32_t sa = 0, pa = 0;
      for (int t = first_tile(false); more(t); t = next_tile(t, false)) {
        const Tile tl = a.down_tiles[t];
        if (tl.b < 0) continue;
        const BlockMeta m = a.meta[tl.b];
#ifdef FFWD_PROBE
        const unsigned long long ct = clock64();
        mbar_wait_sleep(&sm.bar->tempty[acc], acc_phase ^ 1);
        pr.wait_t += clock64() - ct;
#else
        mbar_wait_sleep(&sm.bar->tempty[acc], acc_phase ^ 1);
#endif
        tc_fence_after();
        if constexpr (kSplit)
          mma_tile_split(sm, tmem + acc * BN, m.ktot / BK, idesc, kLbo, 1024, 2048, stage, phase,
                         sa, pa, &pr);
        else
          mma_tile(sm, tmem + acc * BN, m.ktot / BK, idesc, kLbo, 1024, 2048, stage, phase);
        umma_commit(&sm.bar->tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
#ifdef FFWD_PROBE
      if (blockIdx.x < 256) {
        unsigned long long* o = g_probe_down[blockIdx.x];
        o[0] = pr.wait_a; o[1] = pr.wait_b; o[2] = pr.wait_t; o[3] = clock64() - pr.t0;
        o[4] = pr.stages;
      }
#endif
    }
    __syncwarp();
  } else {
    // ---------------- epilogue
    const int ew = warp - kEpiWarp0;
    const int row = ew * 32 + static_cast<int>(lane);
    uint32_t acc = 0, acc_phase = 0;
    for (int t = first_tile(true); more(t); t = next_tile(t, true)) {
      const Tile tl = a.down_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      mbar_wait_sleep(&sm.bar->tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
      const size_t row_off = static_cast<size_t>(m.tok0 + row) * a.d + tl.n0;
      const bool live = row < m.ntok;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t v[16];
        tmem_ld16(tb + c, v);
        tmem_ld_wait();
        if (live && tl.kind != 3) {  // kind 3: pair shadow, no stores
          float o[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = __uint_as_float(v[j]);
          if (a.residual) {  // fused residual add (engine.py:308)
            const float4* res = reinterpret_cast<const float4*>(a.residual + row_off + c);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 r = FFWD_K3_STREAM_EPI ? __ldcs(res + j) : res[j];
              o[4 * j] += r.x;
              o[4 * j + 1] += r.y;
              o[4 * j + 2] += r.z;
              o[4 * j + 3] += r.w;
            }
          }
          if (a.y) {  // null: bf16 output only (a tensor-parallel partial for a bf16 reduce)
            float4* dst = reinterpret_cast<float4*>(a.y + row_off + c);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 v4 = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
              if (FFWD_K3_STREAM_EPI) __stcs(dst + j, v4); else dst[j] = v4;
            }
          }
          if (a.x_next) {  // next layer's bf16 input
            uint4* xn = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.x_next) +
                                                 row_off + c);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint4 v4 = make_uint4(pack_bf16x2(o[8 * j], o[8 * j + 1]),
                                          pack_bf16x2(o[8 * j + 2], o[8 * j + 3]),
                                          pack_bf16x2(o[8 * j + 4], o[8 * j + 5]),
                                          pack_bf16x2(o[8 * j + 6], o[8 * j + 7]));
              if (FFWD_K3_STREAM_EPI) __stcs(xn + j, v4); else xn[j] = v4;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.bar->tempty[acc]);
      if (a.y_done != nullptr && tl.kind == 2) {
        // publish "one more column tile of block b is in Y" to the overlapped TP
        // completion, which reads Y from peer GPUs: system-scope release
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (ew == 0 && lane == 0) {
          __threadfence_system();
          atomicAdd(a.y_done + tl.b, 1u);
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  teardown(sm, warp);
}

template <int BN>
cudaError_t launch_bn(const GemmArgs& a, cudaStream_t s) {
  CUtensorMap th, tw, twt, thh;
  if (encode_tmap_2d_bf16(&th, a.h, a.hcols, static_cast<uint64_t>(a.n_blk) * BM, BK, BM) !=
      CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&thh, a.h, a.hcols, static_cast<uint64_t>(a.n_blk) * BM, BK, BM / 2) !=
      CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&tw, a.wd, a.d, a.wd_rows, 64, 1) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&twt, a.wd, a.d, a.wd_rows, 64, BK) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  CUtensorMap twpf;  // L2 prefetch of whole BN-column row segments
  if (encode_tmap_2d_bf16_sw(&twpf, a.wd, a.d, a.wd_rows, BN, 1, false) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  constexpr size_t smem = smem_bytes<BK * BN * 2>();
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = ensure_smem_limit(down_proj_kernel<BN>, smem, attr); e != cudaSuccess)
    return e;
  int grid = a.num_sms < a.down_cap ? a.num_sms : a.down_cap;
  if constexpr (kPairA) {
    grid &= ~1;  // whole CTA pairs; the plan pads the tile table to pairs
    if (grid < 2) grid = 2;
  }
  return launch_k(down_proj_kernel<BN>, dim3(grid), dim3(kThreads), smem, s, kPairA ? 2 : 1, th,
                  tw, twt, thh, twpf, a);
}

}  // namespace

bool down_proj_paired() { return kPairA; }

cudaError_t launch_down_proj(const GemmArgs& a, cudaStream_t s) {
  switch (a.bn_down) {
    case 256: return launch_bn<256>(a, s);
    case 128: return launch_bn<128>(a, s);
    case 64: return launch_bn<64>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ffwd

#ifdef FFWD_PROBE
extern "C" __attribute__((visibility("default"))) int ffwd_probe_read_down(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, ffwd::g_probe_down, sizeof(ffwd::g_probe_down)) == cudaSuccess ? 0 : 1;
}
#endif
