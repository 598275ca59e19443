// K2 / K3: the sparse SwiGLU FFN as tcgen05 gather-GEMMs (sm_100a).
//
// Layer-major batching: one launch covers every 128-token block
// of a layer.  Each block is a "group" with its own neuron subset, i.e. a
// grouped GEMM with M = 128 tokens per group and a per-group gathered B.
//
//   K2 up_proj_kernel   H_b[:, p] = silu(X_b . Wg[:, idx_b[p]]) * (X_b . Wu[:, idx_b[p]])
//                       (sparse.py:81-91) for p < k_b, plus the compensator hidden
//                       C_b = silu(X_b . Wc1) (compensator.py:52-58) as extra tiles.
//                       A = X_b via 2-D TMA; B = selected rows of the neuron-major
//                       [gate^T | up^T | Wc1^T] via TMA tile::gather4; D in TMEM;
//                       SiLU(gate) * up fused in the TMEM -> register epilogue.
//   K3 down_proj_kernel Y_b = [H_b | C_b] . [W_down[idx_b, :] ; Wc2]
//                       (sparse.py:91 + compensator.py:61-66): the compensator is
//                       simply extra K iterations into the same TMEM accumulator.
//                       A = H_b via 2-D TMA (K-major); B = gathered W_down rows,
//                       MN-major (d contiguous) via tile::gather4.
//
// Both kernels are persistent and warp specialised (TMA producer warp, one MMA
// issuing thread, four epilogue warps), with a STAGES-deep smem ring and a
// double-buffered TMEM accumulator so the epilogue of tile i overlaps the
// main loop of tile i+1.  The tile tables come from plan_kernel on the device,
// so per-(block, rank) ragged k under tensor parallelism needs no host sync.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "ffwd_internal.h"
#include "sm100.cuh"

namespace ffwd {

namespace {

constexpr int BM = 128;       // tokens per tile (one block)
constexpr int BK = 64;        // K per pipeline stage (128 B of bf16 = one swizzle row)
constexpr int UP_BN = 256;    // B rows per up-proj tile: 128 gate + 128 up (or 256 comp)
constexpr int kStages = 4;
constexpr int kThreads = 256;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 epilogue
constexpr uint32_t kTmemCols = 512;

constexpr int kABytes = BM * BK * 2;  // 16 KiB

__host__ __device__ constexpr int round_up(int v, int m) { return (v + m - 1) / m * m; }

struct SmemBarriers {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

template <int kBBytes>
constexpr size_t smem_bytes() {
  return 1024 /*alignment slack*/ + static_cast<size_t>(kStages) * (kABytes + kBBytes) +
         sizeof(SmemBarriers);
}

// ------------------------------------------------------------------ plan
constexpr int kPlanThreads = 256;
constexpr int kMaxGroups = 2048;

// Blocks are ordered dense-first, then predicted; each class is cut into
// groups of `group` blocks and a group's tiles are laid out tile-index-major
// (for i: for block in group), so concurrently running CTAs share the same
// compacted neuron window (L2 reuse of gathered weight rows)
// while the group's X / H blocks stay L2 resident.
__device__ __forceinline__ int order_to_block(int o, int n_dense_lo, const PlanArgs& a) {
  // dense blocks: [0, sparse_begin) and [sparse_begin + sparse_count, n_blk)
  if (o < n_dense_lo) return o;
  const int n_dense = a.n_blk - a.sparse_count;
  if (o < n_dense) return a.sparse_begin + a.sparse_count + (o - n_dense_lo);
  return a.sparse_begin + (o - n_dense);
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(PlanArgs a, BlockMeta* meta,
                                                             Tile* up, int up_cap, Tile* down,
                                                             int down_cap, PlanCounts* pc) {
  __shared__ int s_base[kMaxGroups + 1];
  __shared__ int s_gsz[kMaxGroups];
  __shared__ int s_gmax[kMaxGroups];
  __shared__ int s_ngroups, s_total, s_hcols;
  const int tid = threadIdx.x;
  const int rc64 = round_up(a.rc_local, 64);
  if (tid == 0) s_hcols = 0;
  __syncthreads();
  for (int b = tid; b < a.n_blk; b += kPlanThreads) {
    BlockMeta m;
    m.tok0 = b * kBlockTokens;
    m.ntok = min(kBlockTokens, a.T - m.tok0);
    const bool sparse = b >= a.sparse_begin && b < a.sparse_begin + a.sparse_count;
    if (sparse) {
      const int row = b - a.sparse_begin;
      m.kcount = a.counts ? a.counts[row] : a.k_shared;
      m.idx_row = a.idx_shared ? 0 : row;
      m.comp = (a.has_comp && rc64 > 0) ? rc64 : 0;
    } else {
      m.kcount = a.f_local;
      m.idx_row = -1;
      m.comp = 0;
    }
    m.kpad = round_up(m.kcount, 64);
    m.ktot = m.kpad + m.comp;
    m.n_gu = (m.kcount + 127) / 128;
    meta[b] = m;
    atomicMax(&s_hcols, m.ktot);
  }
  __syncthreads();
  const int n_dense_lo = a.sparse_begin;
  const int n_dense = a.n_blk - a.sparse_count;

  // ---- up-projection tile table
  if (tid == 0) {
    int g = 0, base = 0;
    for (int cls = 0; cls < 2; ++cls) {
      const int o_lo = cls == 0 ? 0 : n_dense, o_hi = cls == 0 ? n_dense : a.n_blk;
      for (int o = o_lo; o < o_hi && g < kMaxGroups; o += a.up_group) {
        const int sz = min(a.up_group, o_hi - o);
        int mx = 0;
        for (int j = 0; j < sz; ++j) {
          const BlockMeta& m = meta[order_to_block(o + j, n_dense_lo, a)];
          mx = max(mx, m.n_gu + (m.comp + UP_BN - 1) / UP_BN);
        }
        s_base[g] = base;
        s_gsz[g] = sz;
        s_gmax[g] = o;  // first order index of the group (reused below)
        base += mx * sz;
        ++g;
      }
    }
    s_base[g] = base;
    s_ngroups = g;
    s_total = min(base, up_cap);
  }
  __syncthreads();
  for (int slot = tid; slot < s_total; slot += kPlanThreads) {
    int lo = 0, hi = s_ngroups - 1;  // last group with base <= slot
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_base[mid] <= slot) lo = mid; else hi = mid - 1;
    }
    const int rel = slot - s_base[lo], sz = s_gsz[lo];
    const int i = rel / sz, b = order_to_block(s_gmax[lo] + rel % sz, n_dense_lo, a);
    const BlockMeta m = meta[b];
    Tile t{-1, 0, 0, 0};
    if (i < m.n_gu) {
      t = Tile{b, i * 128, 0, 0};
    } else if (i < m.n_gu + (m.comp + UP_BN - 1) / UP_BN) {
      t = Tile{b, (i - m.n_gu) * UP_BN, 1, 0};
    }
    up[slot] = t;
  }
  __syncthreads();

  // ---- down-projection tile table: groups of down_group blocks, column-tile major
  const int nt = a.d / a.bn_down;
  const int total_down = min(a.n_blk * nt, down_cap);
  for (int slot = tid; slot < total_down; slot += kPlanThreads) {
    const int g = slot / (a.down_group * nt);
    const int o0 = g * a.down_group;
    const int sz = min(a.down_group, a.n_blk - o0);
    const int rel = slot - o0 * nt;
    const int j = rel / sz, o = o0 + rel % sz;
    down[slot] = Tile{order_to_block(o, n_dense_lo, a), j * a.bn_down, 2, 0};
  }
  if (tid == 0) {
    pc->n_up = s_total;
    pc->n_down = total_down;
    pc->hcols = s_hcols;
  }
}

// ------------------------------------------------------------------ common pieces
template <int kBBytes>
struct Smem {
  uint8_t* a;
  uint8_t* b;
  SmemBarriers* bar;
  __device__ Smem(uint8_t* raw) {
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) &
                                               ~uintptr_t(1023));
    a = base;
    b = base + kStages * kABytes;
    bar = reinterpret_cast<SmemBarriers*>(b + kStages * kBBytes);
  }
  __device__ uint8_t* a_stage(int s) const { return a + s * kABytes; }
  __device__ uint8_t* b_stage(int s) const { return b + s * kBBytes; }
};

template <int kBBytes>
__device__ __forceinline__ void kernel_prologue(Smem<kBBytes>& sm, int warp) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.bar->full[i], 1);
      mbar_init(&sm.bar->empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.bar->tfull[i], 1);
      mbar_init(&sm.bar->tempty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(&sm.bar->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

template <int kBBytes>
__device__ __forceinline__ void kernel_epilogue(Smem<kBBytes>& sm, int warp) {
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<kTmemCols>(sm.bar->tmem_base);
}

__device__ __forceinline__ int neuron_at(const BlockMeta& m, const int32_t* __restrict__ idx,
                                         int ld_idx, int p) {
  if (p >= m.kcount) return 0;  // padding row: contributes to masked / zero columns only
  return m.idx_row < 0 ? p : __ldg(idx + static_cast<size_t>(m.idx_row) * ld_idx + p);
}

// MMA issue loop shared by both kernels: one elected thread, 4 UMMA_K=16 steps per stage.
template <int kBBytes>
__device__ __forceinline__ void mma_tile(Smem<kBBytes>& sm, uint32_t tmem_d, int nk,
                                         uint32_t idesc, uint32_t b_lbo, uint32_t b_sbo,
                                         uint32_t b_kstep, uint32_t& stage, uint32_t& phase) {
  for (int kb = 0; kb < nk; ++kb) {
    mbar_wait(&sm.bar->full[stage], phase);
    tc_fence_after();
    if (elect_one()) {
      const uint64_t adesc = make_sdesc_sw128(smem_u32(sm.a_stage(stage)), 16, 1024);
      const uint64_t bdesc = make_sdesc_sw128(smem_u32(sm.b_stage(stage)), b_lbo, b_sbo);
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        umma_bf16(tmem_d, adesc + static_cast<uint64_t>(2 * kk),
                  bdesc + static_cast<uint64_t>((b_kstep >> 4) * kk), idesc,
                  (kb | kk) != 0 ? 1u : 0u);
      }
      umma_commit(&sm.bar->empty[stage]);
    }
    __syncwarp();
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// ------------------------------------------------------------------ K2
constexpr int kUpBBytes = UP_BN * BK * 2;  // 32 KiB

__global__ void __launch_bounds__(kThreads, 1)
    up_proj_kernel(const __grid_constant__ CUtensorMap tm_x,
                   const __grid_constant__ CUtensorMap tm_w, GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  Smem<kUpBBytes> sm(smem_raw);
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w);
  }
  kernel_prologue(sm, warp);
  const uint32_t tmem = sm.bar->tmem_base;
  const int n_tiles = a.counts->n_up;
  const int nk = a.d / BK;

  if (warp == 0) {
    // ---------------- TMA producer: lane l gathers B rows [8l, 8l+8) of each stage
    const uint64_t pol_x = policy_evict_last();
    const uint64_t pol_w = policy_evict_normal();
    uint32_t stage = 0, phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = a.up_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      int rows[8];
      if (tl.kind == 0) {
        const int half = lane >> 4;
        const int p0 = tl.n0 + (lane & 15) * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          rows[i] = neuron_at(m, a.idx, a.ld_idx, p0 + i) + half * a.f_local;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) rows[i] = 2 * a.f_local + tl.n0 + lane * 8 + i;
      }
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&sm.bar->empty[stage], phase ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&sm.bar->full[stage], kABytes + kUpBBytes);
          tma_load_2d(&tm_x, &sm.bar->full[stage], sm.a_stage(stage), kb * BK, m.tok0, pol_x);
        }
        uint8_t* dst = sm.b_stage(stage) + lane * 8 * 128;
        tma_gather4(&tm_w, &sm.bar->full[stage], dst, kb * BK, rows[0], rows[1], rows[2],
                    rows[3], pol_w);
        tma_gather4(&tm_w, &sm.bar->full[stage], dst + 512, kb * BK, rows[4], rows[5],
                    rows[6], rows[7], pol_w);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = make_idesc_bf16(BM, UP_BN, false, false);
    uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = a.up_tiles[t];
      if (tl.b < 0) continue;
      mbar_wait(&sm.bar->tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      mma_tile(sm, tmem + acc * UP_BN, nk, idesc, 16, 1024, 32, stage, phase);
      if (elect_one()) umma_commit(&sm.bar->tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> regs -> SiLU(g)*u -> bf16 H
    const int ew = warp - 4;
    const int row = ew * 32 + static_cast<int>(lane);
    uint32_t acc = 0, acc_phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = a.up_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      mbar_wait(&sm.bar->tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem + acc * UP_BN + (static_cast<uint32_t>(ew * 32) << 16);
      __nv_bfloat16* hrow = static_cast<__nv_bfloat16*>(a.h) +
                            static_cast<size_t>(tl.b * kBlockTokens + row) * a.hcols;
      if (tl.kind == 0) {
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          const int pos = tl.n0 + c;
          if (pos >= m.kpad) break;
          uint32_t g[32], u[32];
          tmem_ld32(tb + c, g);
          tmem_ld32(tb + 128 + c, u);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float h0 = silu_f32(__uint_as_float(g[2 * j])) * __uint_as_float(u[2 * j]);
            float h1 = silu_f32(__uint_as_float(g[2 * j + 1])) * __uint_as_float(u[2 * j + 1]);
            if (pos + 2 * j >= m.kcount) h0 = 0.0f;
            if (pos + 2 * j + 1 >= m.kcount) h1 = 0.0f;
            packed[j] = pack_bf16x2(h0, h1);
          }
          uint4* dst = reinterpret_cast<uint4*>(hrow + pos);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[j] = make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2],
                                packed[4 * j + 3]);
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < UP_BN; c += 32) {
          const int col = tl.n0 + c;
          if (col >= m.comp) break;
          uint32_t g[32];
          tmem_ld32(tb + c, g);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            packed[j] = pack_bf16x2(silu_f32(__uint_as_float(g[2 * j])),
                                    silu_f32(__uint_as_float(g[2 * j + 1])));
          uint4* dst = reinterpret_cast<uint4*>(hrow + m.kpad + col);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[j] = make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2],
                                packed[4 * j + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.bar->tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  kernel_epilogue(sm, warp);
}

// ------------------------------------------------------------------ K3
template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    down_proj_kernel(const __grid_constant__ CUtensorMap tm_h,
                     const __grid_constant__ CUtensorMap tm_w, GemmArgs a) {
  constexpr int kBBytes = BK * BN * 2;
  constexpr int kChunks = BN / 64;          // 64-column (128 B) atoms along N
  constexpr uint32_t kLbo = (BK / 8) * 1024;  // MN-direction atom stride
  extern __shared__ uint8_t smem_raw[];
  Smem<kBBytes> sm(smem_raw);
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_h);
    tma_prefetch_desc(&tm_w);
  }
  kernel_prologue(sm, warp);
  const uint32_t tmem = sm.bar->tmem_base;
  const int n_tiles = a.counts->n_down;

  if (warp == 0) {
    // ---------------- TMA producer: 16 row-quads x kChunks column atoms per stage
    const uint64_t pol_h = policy_evict_last();
    const uint64_t pol_w = policy_evict_normal();
    constexpr int kPerLane = (16 * kChunks + 31) / 32;
    uint32_t stage = 0, phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = a.down_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      const int nk = m.ktot / BK;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&sm.bar->empty[stage], phase ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&sm.bar->full[stage], kABytes + kBBytes);
          tma_load_2d(&tm_h, &sm.bar->full[stage], sm.a_stage(stage), kb * BK,
                      tl.b * kBlockTokens, pol_h);
        }
#pragma unroll
        for (int q = 0; q < kPerLane; ++q) {
          const int job = static_cast<int>(lane) + 32 * q;
          if (job >= 16 * kChunks) break;
          const int quad = job & 15, chunk = job >> 4;
          int r[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int p = kb * BK + quad * 4 + i;
            r[i] = p < m.kpad ? neuron_at(m, a.idx, a.ld_idx, p) : a.f_local + (p - m.kpad);
          }
          uint8_t* dst = sm.b_stage(stage) + chunk * kLbo + (quad >> 1) * 1024 + (quad & 1) * 512;
          tma_gather4(&tm_w, &sm.bar->full[stage], dst, tl.n0 + chunk * 64, r[0], r[1], r[2],
                      r[3], pol_w);
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16(BM, BN, false, true);
    uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = a.down_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      mbar_wait(&sm.bar->tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      mma_tile(sm, tmem + acc * BN, m.ktot / BK, idesc, kLbo, 1024, 2048, stage, phase);
      if (elect_one()) umma_commit(&sm.bar->tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int row = ew * 32 + static_cast<int>(lane);
    uint32_t acc = 0, acc_phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = a.down_tiles[t];
      if (tl.b < 0) continue;
      const BlockMeta m = a.meta[tl.b];
      mbar_wait(&sm.bar->tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
      const size_t row_off = static_cast<size_t>(m.tok0 + row) * a.d + tl.n0;
      float* yrow = a.y + row_off;
      const bool live = row < m.ntok;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tmem_ld32(tb + c, v);
        tmem_ld_wait();
        if (live) {
          float o[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __uint_as_float(v[j]);
          if (a.residual) {  // fused residual add (engine.py:308)
            const float4* res = reinterpret_cast<const float4*>(a.residual + row_off + c);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 r = res[j];
              o[4 * j] += r.x;
              o[4 * j + 1] += r.y;
              o[4 * j + 2] += r.z;
              o[4 * j + 3] += r.w;
            }
          }
          float4* dst = reinterpret_cast<float4*>(yrow + c);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
          if (a.x_next) {  // next layer's bf16 input, written once here
            uint4* xn = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.x_next) +
                                                 row_off + c);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              xn[j] = make_uint4(pack_bf16x2(o[8 * j], o[8 * j + 1]),
                                 pack_bf16x2(o[8 * j + 2], o[8 * j + 3]),
                                 pack_bf16x2(o[8 * j + 4], o[8 * j + 5]),
                                 pack_bf16x2(o[8 * j + 6], o[8 * j + 7]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.bar->tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  kernel_epilogue(sm, warp);
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

}  // namespace

CUresult encode_tmap_2d_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                             uint32_t box_inner, uint32_t box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) return CUDA_ERROR_NOT_FOUND;
  const cuuint64_t dims[2] = {inner, rows};
  const cuuint64_t strides[1] = {inner * 2};
  const cuuint32_t box[2] = {box_inner, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

cudaError_t launch_plan(const PlanArgs& a, BlockMeta* meta, Tile* up_tiles, int up_cap,
                        Tile* down_tiles, int down_cap, PlanCounts* counts, cudaStream_t s) {
  plan_kernel<<<1, kPlanThreads, 0, s>>>(a, meta, up_tiles, up_cap, down_tiles, down_cap,
                                         counts);
  return cudaGetLastError();
}

cudaError_t launch_up_proj(const GemmArgs& a, cudaStream_t s) {
  CUtensorMap tx, tw;
  if (encode_tmap_2d_bf16(&tx, a.x, a.d, a.T, BK, BM) != CUDA_SUCCESS) return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&tw, a.wgu_t, a.d, a.wgu_rows, BK, 1) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  constexpr size_t smem = smem_bytes<kUpBBytes>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(up_proj_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = a.num_sms < a.up_cap ? a.num_sms : a.up_cap;
  up_proj_kernel<<<grid, kThreads, smem, s>>>(tx, tw, a);
  return cudaGetLastError();
}

template <int BN>
static cudaError_t launch_down_bn(const GemmArgs& a, cudaStream_t s) {
  CUtensorMap th, tw;
  if (encode_tmap_2d_bf16(&th, a.h, a.hcols, static_cast<uint64_t>(a.n_blk) * BM, BK, BM) !=
      CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (encode_tmap_2d_bf16(&tw, a.wd, a.d, a.wd_rows, 64, 1) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  constexpr size_t smem = smem_bytes<BK * BN * 2>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(down_proj_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = a.num_sms < a.down_cap ? a.num_sms : a.down_cap;
  down_proj_kernel<BN><<<grid, kThreads, smem, s>>>(th, tw, a);
  return cudaGetLastError();
}

cudaError_t launch_down_proj(const GemmArgs& a, cudaStream_t s) {
  switch (a.bn_down) {
    case 256: return launch_down_bn<256>(a, s);
    case 128: return launch_down_bn<128>(a, s);
    case 64: return launch_down_bn<64>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ffwd
