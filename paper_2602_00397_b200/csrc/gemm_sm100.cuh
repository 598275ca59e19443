// Shared pieces of the two persistent tcgen05 gather-GEMMs (up_proj.cu, down_proj.cu).
//
// CTA layout (P = kProducerWarps, one CTA per SM):
//   warps 0..P-1   TMA producers: each owns 1/P of every stage's B rows and issues
//                  them with tile::gather4 from one lane (row ids staged in shared
//                  memory so every TMA operand is warp-uniform); warp 0 also loads
//                  the A tile.  gather4 throughput is set by the number of issuing
//                  warps (tools/tma_bench.cu), hence several producer warps.  The
//                  full barrier of a stage expects one arrive.expect_tx per warp.
//   warps P..P+3   epilogue: warp P+i reads TMEM lanes [32i, 32i+32) (tile rows).
//   warp P+4       TMEM allocator + the single MMA-issuing thread.
// Pipelines: kStages-deep smem ring (full/empty mbarriers) between producers
// and MMA; two TMEM accumulators (tfull/tempty) between MMA and epilogue, so
// the epilogue of tile i overlaps the main loop of tile i+1.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ffwd_internal.h"
#include "sm100.cuh"

namespace ffwd {
namespace gemm {
// Each kernel TU picks its own producer-warp count (FFWD_PRODUCER_WARPS before the
// include), so everything here has internal linkage.
namespace {

constexpr int BM = 128;           // tokens per tile (one block)
constexpr int BK = 64;             // K per stage: 64 bf16 = one 128 B swizzle row
constexpr int kStages = 4;
// Split rings (FFWD_SPLIT_RING): the gathered B operand gets a deeper ring than the
// 2-D A tile, which a dedicated warp loads on its own barriers.  The gathers' fill
// latency is what the ring has to cover, and a shallower A ring frees the smem.
#ifdef FFWD_SPLIT_RING
constexpr bool kSplit = true;
constexpr int kStagesA = FFWD_STAGES_A;
constexpr int kStagesB = FFWD_STAGES_B;
#else
constexpr bool kSplit = false;
constexpr int kStagesA = kStages;
constexpr int kStagesB = kStages;
#endif
// CTA pairs (FFWD_PAIR_A, split rings only): the two CTAs of a cluster work on two
// neuron tiles of the same token block at the same time and each loads half of the
// shared A tile, multicast to both; both MMAs release every A slot in both CTAs.
#ifdef FFWD_PAIR_A
constexpr bool kPairA = true;
#else
constexpr bool kPairA = false;
#endif
#ifndef FFWD_PRODUCER_WARPS
#define FFWD_PRODUCER_WARPS 8
#endif
constexpr int kProducerWarps = FFWD_PRODUCER_WARPS;  // TMA gather4 issue rate scales with warps
constexpr int kEpiWarp0 = kProducerWarps;            // multiple of 4: warp % 4 = TMEM lane quadrant
constexpr int kMmaWarp = kProducerWarps + 4;
constexpr int kAWarp = kProducerWarps + 5;  // A loader (split rings only)
// Dynamic tile claiming (FFWD_DYN_TILES, per kernel TU; TileQueue below)
#ifdef FFWD_DYN_TILES
constexpr bool kDyn = true;
#else
constexpr bool kDyn = false;
#endif
// warps reading the tile queue: all roles but producer warp 0, which claims
constexpr int kTileConsumers = kProducerWarps + 4 + (kSplit ? 1 : 0);
constexpr int kThreads = (kProducerWarps + 5 + (kSplit ? 1 : 0)) * 32;
static_assert(kProducerWarps % 4 == 0 && 64 % kProducerWarps == 0, "producer split");
constexpr uint32_t kTmemCols = 512;
// FFWD_A_LDGSTS (per kernel TU): the A tile is copied by the A-loader warp's 32 lanes with
// 16 B cp.async (the LSU path) instead of one TMA box, so A does not queue in the SM's TMA
// unit behind the B gathers; fullA then counts one cp.async arrival per lane.
#ifdef FFWD_A_LDGSTS
constexpr bool kALdgsts = true;
constexpr uint32_t kALanes = 32;
#else
constexpr bool kALdgsts = false;
constexpr uint32_t kALanes = 1;
#endif
// FFWD_B_LDGSTS (per kernel TU, K3 only): the gathered B rows are copied by every producer
// lane with 16 B cp.async into the 128B-swizzled layout instead of TMA tile::gather4, so
// the row gathers bypass the SM's TMA unit; full[] then counts one arrival per lane.
#ifdef FFWD_B_LDGSTS
constexpr bool kBLdgsts = true;
constexpr uint32_t kBLanes = 32;
#else
constexpr bool kBLdgsts = false;
constexpr uint32_t kBLanes = 1;
#endif
constexpr int kABytes = BM * BK * 2;  // 16 KiB

__host__ __device__ constexpr int round_up(int v, int m) { return (v + m - 1) / m * m; }

// rows gathered per stage: the up projection gathers its 256 B-operand rows, the down
// projection its 64 K rows (FFWD_GATHER_ROWS; smaller row staging leaves K3 room for a
// co-resident CTA of the overlapped TP completion)
#ifndef FFWD_GATHER_ROWS
#define FFWD_GATHER_ROWS 256
#endif
constexpr int kGatherRows = FFWD_GATHER_ROWS;

// Dynamic tile claiming: producer warp 0 claims the CTA's next tile from a global counter
// (atomicAdd, table order) when it is about to start it, and hands the id to the CTA's
// other roles through a small shared-memory queue, so every role walks the same
// sequence.  A CTA thus takes a tile exactly when its gathers are ready for one: the long
// tiles (dense blocks) and the last wave no longer set the kernel's end as with static
// striding.  Each tile's arithmetic is unchanged (results are bit-identical).
constexpr int kTQ = 4;
struct TileQueue {
  uint64_t full[kTQ];
  uint64_t empty[kTQ];  // one arrival per consuming warp
  int tile[kTQ];
};

__device__ __forceinline__ void tq_init(TileQueue* q, uint32_t consumers) {
  for (int i = 0; i < kTQ; ++i) {
    mbar_init(&q->full[i], 1);
    mbar_init(&q->empty[i], consumers);
  }
}

// Cluster-scope acquire wait (the peer CTA posted the slot with a remote release-arrive).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void st_shared_remote(int* p, uint32_t rank, int v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(remote), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

struct TileCursor {
  uint32_t i = 0, ph = 0;
  // Consumers: the next tile id (-1 = no more).  `warp_wide`: every lane of the warp
  // calls it (lane 0 releases the slot after the warp read it); else a single thread.
  __device__ __forceinline__ int next(TileQueue* q, bool warp_wide) {
    mbar_wait(&q->full[i], ph);
    const int t = q->tile[i];
    if (warp_wide) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&q->empty[i]);
    } else {
      mbar_arrive(&q->empty[i]);
    }
    advance();
    return t;
  }
  // The claiming warp (all lanes): claims the next tile, posts it, returns it.
  __device__ __forceinline__ int claim(TileQueue* q, int* counter, int n_tiles) {
    int t = 0;
    if ((threadIdx.x & 31) == 0) {
      mbar_wait(&q->empty[i], ph ^ 1);
      t = atomicAdd(counter, 1);
      if (t >= n_tiles) t = -1;
      q->tile[i] = t;
      mbar_arrive(&q->full[i]);
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    advance();
    return t;
  }
  // CTA pairs (the two CTAs of a cluster run table slots 2p and 2p + 1 together): rank 0's
  // producer warp 0 claims a pair index p and posts it into both CTAs' queues; every
  // consumer of either CTA releases the slot on rank 0's queue (its empty barrier counts
  // both CTAs' consumers).  Returns this CTA's slot 2p + rank (-1 = no more).
  __device__ __forceinline__ int claim_pair(TileQueue* q, int* counter, int n_tiles) {
    int p = 0;
    if ((threadIdx.x & 31) == 0) {
      mbar_wait_cluster(&q->empty[i], ph ^ 1);
      p = atomicAdd(counter, 1);
      if (2 * p >= n_tiles) p = -1;
      q->tile[i] = p;
      st_shared_remote(&q->tile[i], 1, p);
      mbar_arrive(&q->full[i]);
      mbar_arrive_remote(&q->full[i], 1);
    }
    p = __shfl_sync(0xffffffffu, p, 0);
    advance();
    return p < 0 ? -1 : 2 * p;
  }
  __device__ __forceinline__ int next_pair(TileQueue* q, bool warp_wide, uint32_t rank) {
    mbar_wait_cluster(&q->full[i], ph);
    const int p = q->tile[i];
    if (warp_wide) __syncwarp();
    if (!warp_wide || (threadIdx.x & 31) == 0) {
      if (rank == 0) mbar_arrive(&q->empty[i]);
      else mbar_arrive_remote(&q->empty[i], 0);
    }
    advance();
    return p < 0 ? -1 : 2 * p + static_cast<int>(rank);
  }
  __device__ __forceinline__ void advance() {
    if (++i == kTQ) {
      i = 0;
      ph ^= 1;
    }
  }
};

struct Barriers {
  uint64_t full[kStagesB];   // B (and, unsplit, A) landed
  uint64_t empty[kStagesB];
  uint64_t fullA[kStagesA];  // split rings: A landed / A slot free
  uint64_t emptyA[kStagesA];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  uint32_t pad;
  TileQueue q;  // dynamic tile claiming only
  alignas(16) int rows[kProducerWarps][kGatherRows / kProducerWarps];  // gather row ids (int4)
};

template <int kBBytes>
constexpr size_t smem_bytes() {
  return 1024 + static_cast<size_t>(kStagesA) * kABytes + static_cast<size_t>(kStagesB) * kBBytes +
         sizeof(Barriers);
}

template <int kBBytes>
struct Smem {
  uint8_t* a;
  uint8_t* b;
  Barriers* bar;
  __device__ explicit Smem(uint8_t* raw) {
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) &
                                               ~uintptr_t(1023));
    a = base;
    b = base + kStagesA * kABytes;
    bar = reinterpret_cast<Barriers*>(b + kStagesB * kBBytes);
  }
  __device__ uint8_t* a_stage(int s) const { return a + s * kABytes; }
  __device__ uint8_t* b_stage(int s) const { return b + s * kBBytes; }
};

template <int kBBytes>
__device__ __forceinline__ void prologue(Smem<kBBytes>& sm, int warp) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStagesB; ++i) {
      mbar_init(&sm.bar->full[i], kProducerWarps * kBLanes);
      mbar_init(&sm.bar->empty[i], 1);
    }
    for (int i = 0; i < kStagesA; ++i) {
      mbar_init(&sm.bar->fullA[i], kALanes);
      mbar_init(&sm.bar->emptyA[i], kPairA ? 2 : 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.bar->tfull[i], 1);
      mbar_init(&sm.bar->tempty[i], 128);
    }
    // pairs: rank 0's empty barriers count both CTAs' consumers (the peer's warp 0 too)
    if constexpr (kDyn) tq_init(&sm.bar->q, kPairA ? 2 * kTileConsumers + 1 : kTileConsumers);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<kTmemCols>(&sm.bar->tmem_base);
  tc_fence_before();
  __syncthreads();
  if constexpr (kPairA) cluster_sync_all();  // peers' barriers initialised before any multicast
  tc_fence_after();
}

template <int kBBytes>
__device__ __forceinline__ void teardown(Smem<kBBytes>& sm, int warp) {
  tc_fence_before();
  __syncthreads();
  if constexpr (kPairA) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<kTmemCols>(sm.bar->tmem_base);
}

// Neuron id at compacted position p of a block; positions past kcount map to
// row 0 (their products land in columns that are masked or multiplied by 0).
__device__ __forceinline__ int neuron_at(const BlockMeta& m, const int32_t* __restrict__ idx,
                                         int ld_idx, int p) {
  if (p >= m.kcount) return 0;
  return m.idx_row < 0 ? p : __ldg(idx + static_cast<size_t>(m.idx_row) * ld_idx + p);
}

// Single elected thread: 4 UMMA_K=16 MMAs per stage, then release the stage.
template <int kBBytes>
__device__ __forceinline__ void mma_tile(Smem<kBBytes>& sm, uint32_t tmem_d, int nk,
                                         uint32_t idesc, uint32_t b_lbo, uint32_t b_sbo,
                                         uint32_t b_kstep, uint32_t& stage, uint32_t& phase) {
  for (int kb = 0; kb < nk; ++kb) {
    mbar_wait(&sm.bar->full[stage], phase);
    tc_fence_after();
    const uint64_t adesc = make_sdesc_sw128(smem_u32(sm.a_stage(stage)), 16, 1024);
    const uint64_t bdesc = make_sdesc_sw128(smem_u32(sm.b_stage(stage)), b_lbo, b_sbo);
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      umma_bf16(tmem_d, adesc + static_cast<uint64_t>(2 * kk),
                bdesc + static_cast<uint64_t>((b_kstep >> 4) * kk), idesc,
                (kb | kk) != 0 ? 1u : 0u);
    }
    umma_commit(&sm.bar->empty[stage]);
    if (++stage == kStagesB) {
      stage = 0;
      phase ^= 1;
    }
  }
}

template <int N>
__device__ __forceinline__ void advance_n(uint32_t& stage, uint32_t& phase) {
  if (++stage == N) {
    stage = 0;
    phase ^= 1;
  }
}

__device__ __forceinline__ void advance(uint32_t& stage, uint32_t& phase) {
  advance_n<kStagesB>(stage, phase);
}

// Split rings: the MMA waits for the stage's A slot and B slot separately and
// releases both.
// FFWD_PROBE builds (timing experiments only): the MMA thread's cycles spent waiting
// for A and for B, accumulated per CTA.
struct Probe {
  unsigned long long wait_a = 0, wait_b = 0, wait_t = 0, t0 = 0, stages = 0;
};

template <int kBBytes>
__device__ __forceinline__ void mma_tile_split(Smem<kBBytes>& sm, uint32_t tmem_d, int nk,
                                               uint32_t idesc, uint32_t b_lbo, uint32_t b_sbo,
                                               uint32_t b_kstep, uint32_t& sb, uint32_t& pb,
                                               uint32_t& sa, uint32_t& pa,
                                               Probe* pr = nullptr) {
  for (int kb = 0; kb < nk; ++kb) {
#ifdef FFWD_PROBE
    const unsigned long long c0 = clock64();
    mbar_wait(&sm.bar->fullA[sa], pa);
    const unsigned long long c1 = clock64();
    mbar_wait(&sm.bar->full[sb], pb);
    const unsigned long long c2 = clock64();
    if (pr) {
      pr->wait_a += c1 - c0;
      pr->wait_b += c2 - c1;
      pr->stages += 1;
    }
#else
    mbar_wait(&sm.bar->fullA[sa], pa);
    mbar_wait(&sm.bar->full[sb], pb);
#endif
    if constexpr (kALdgsts || kBLdgsts) fence_proxy_async_smem();  // cp.async (generic) -> UMMA
    tc_fence_after();
    const uint64_t adesc = make_sdesc_sw128(smem_u32(sm.a_stage(sa)), 16, 1024);
    const uint64_t bdesc = make_sdesc_sw128(smem_u32(sm.b_stage(sb)), b_lbo, b_sbo);
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      umma_bf16(tmem_d, adesc + static_cast<uint64_t>(2 * kk),
                bdesc + static_cast<uint64_t>((b_kstep >> 4) * kk), idesc,
                (kb | kk) != 0 ? 1u : 0u);
    }
    umma_commit(&sm.bar->empty[sb]);
    if constexpr (kPairA)
      umma_commit_mc(&sm.bar->emptyA[sa], 0x3);  // both CTAs' A slot sa is free of this MMA
    else
      umma_commit(&sm.bar->emptyA[sa]);
    advance_n<kStagesB>(sb, pb);
    advance_n<kStagesA>(sa, pa);
  }
}

}  // namespace
}  // namespace gemm
}  // namespace ffwd
