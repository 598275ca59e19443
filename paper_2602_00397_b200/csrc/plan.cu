// Device-side tile planning for the up / down gather-GEMMs (a few CTAs: each recomputes
// the per-block prefix and writes a strided share of the tile slots).
//
// Reads the per-block neuron counts the top-k kernel produced (ragged under
// tensor parallelism) and writes the block descriptors plus both persistent
// kernels' tile tables, so no host synchronisation sits between the
// predictor and the FFN GEMMs.
//
// Rasterisation: blocks are ordered dense-first, then predicted; each class
// is cut into groups of `group` blocks, and a group's tiles are laid out
// tile-index-major (for i: for block in group).  Concurrently running CTAs
// therefore share the same compacted neuron window -- the selected indices
// are ascending, so compacted tile i of every block covers about the same
// neuron range -- while the group's X / H blocks stay L2 resident.
#include <cuda_runtime.h>

#include "ffwd_internal.h"
#include "launch.cuh"

namespace ffwd {

namespace {

#ifndef FFWD_MERGE_DENSE
#define FFWD_MERGE_DENSE 1
#endif
#ifndef FFWD_PLAN_BESIDE_TOPK
#define FFWD_PLAN_BESIDE_TOPK 1
#endif
constexpr int kPlanThreads = 512;
constexpr int kMaxBlocks = 4096;
constexpr int kUpBN = 256;  // rows per compensator up-projection tile

__host__ __device__ constexpr int rup(int v, int m) { return (v + m - 1) / m * m; }

__device__ __forceinline__ int order_to_block(int o, const PlanArgs& a) {
  const int n_lo = a.sparse_begin;                // dense blocks before the predicted range
  const int n_dense = a.n_blk - a.sparse_count;
  if (o < n_lo) return o;
  if (o < n_dense) return a.sparse_begin + a.sparse_count + (o - n_lo);
  return a.sparse_begin + (o - n_dense);
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(PlanArgs a, BlockMeta* meta,
                                                             Tile* up, int up_cap, Tile* down,
                                                             int down_cap, PlanCounts* pc) {
  __shared__ short s_nup[kMaxBlocks];   // up tiles per block, in raster order
  __shared__ short s_ngu[kMaxBlocks];   // of which gate/up tiles
  __shared__ int s_gbase[kMaxBlocks + 1];
  __shared__ int s_hcols;
  __shared__ int s_q, s_dp, s_dn;  // merged dense group: rows, dense pairs, dense tiles
  // Without per-block counts (no tensor parallelism) the plan does not read the top-k's
  // output, so it runs beside the top-k kernel and waits for it only before exiting: the
  // up projection's wait on the plan then still covers the indices.  Every earlier kernel
  // of the layer waited for its predecessor before releasing its dependents, so the
  // previous layer's GEMMs (which read these tables) are complete when this one starts.
  if (a.counts || !FFWD_PLAN_BESIDE_TOPK) pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int rc64 = rup(a.rc_local, 64);
  if (tid == 0) s_hcols = 0;
  __syncthreads();
  for (int o = tid; o < a.n_blk; o += kPlanThreads) {
    const int b = order_to_block(o, a);
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
    m.kpad = rup(m.kcount, 64);
    m.ktot = m.kpad + m.comp;
    m.n_gu = (m.kcount + 127) / 128;
    const int nup = m.n_gu + (m.comp + kUpBN - 1) / kUpBN;
    m.n_up = a.pair_up ? rup(nup, 2) : nup;
    if (blockIdx.x == 0) {
      meta[b] = m;
      if (a.blk_done) a.blk_done[b] = 0;
    }
    s_ngu[o] = static_cast<short>(m.n_gu);
    s_nup[o] = static_cast<short>(nup);
    atomicMax(&s_hcols, m.ktot);
  }
  __syncthreads();

  // Up-projection raster groups.  Predicted blocks: groups of up_group blocks,
  // tile-index-major.  The dense blocks (first / last) join the first predicted group
  // (FFWD_MERGE_DENSE, CTA pairs only): their tile pairs are spread over that group's
  // tile-pair rows in neuron order, so a dense tile reads the W_gu rows the predicted
  // tiles of the same row read (at 50% keep, dense tiles 2p, 2p+1 cover the neurons of
  // predicted tile p) -- one sweep of the weights for both instead of a separate dense
  // group that reads all of W_gu once more.  Otherwise the dense blocks form their own
  // groups (groups never straddle the dense / predicted boundary).
  const int n_dense = a.n_blk - a.sparse_count;
  const bool merge = FFWD_MERGE_DENSE && a.pair_up && n_dense > 0 && a.sparse_count > 0;
  const int g_dense = merge ? 0 : (n_dense + a.up_group - 1) / a.up_group;
  const int sz0 = min(a.up_group, a.sparse_count);  // predicted blocks of the merged group
  const int g_total = merge ? 1 + (a.sparse_count - sz0 + a.up_group - 1) / a.up_group
                            : g_dense + (a.sparse_count + a.up_group - 1) / a.up_group;
  // order range of group g (the merged group 0 spans the dense blocks and sz0 predicted)
  auto group_range = [&](int g, int& o0, int& o1) {
    if (merge) {
      o0 = g == 0 ? 0 : n_dense + sz0 + (g - 1) * a.up_group;
      o1 = g == 0 ? n_dense + sz0 : min(a.n_blk, o0 + a.up_group);
    } else {
      o0 = g < g_dense ? g * a.up_group : n_dense + (g - g_dense) * a.up_group;
      o1 = min(g < g_dense ? n_dense : a.n_blk, o0 + a.up_group);
    }
  };
  // per-group slot counts (max tiles in the group x group size)
  for (int g = tid; g < g_total; g += kPlanThreads) {
    int o0, o1;
    group_range(g, o0, o1);
    if (merge && g == 0) {
      int mxp = 0, dn = 0;
      for (int o = n_dense; o < o1; ++o) mxp = max(mxp, static_cast<int>(s_nup[o]));
      for (int o = 0; o < n_dense; ++o) dn = max(dn, static_cast<int>(s_nup[o]));
      s_q = max(1, rup(mxp, 2) / 2);  // tile-pair rows of the group
      s_dp = (dn + 1) / 2;            // tile pairs per dense block
      s_dn = dn;
      s_gbase[1] = 2 * sz0 * s_q + 2 * n_dense * s_dp;
      continue;
    }
    int mx = 0;
    for (int o = o0; o < o1; ++o) mx = max(mx, static_cast<int>(s_nup[o]));
    if (a.pair_up) mx = rup(mx, 2);  // paired up-projection: whole (i, i+1) tile pairs
    s_gbase[g + 1] = mx * (o1 - o0);
  }
  __syncthreads();
  if (tid == 0) {
    s_gbase[0] = 0;
    for (int g = 0; g < g_total; ++g) s_gbase[g + 1] += s_gbase[g];
  }
  __syncthreads();
  const int total_up = min(s_gbase[g_total], up_cap);
  for (int slot = blockIdx.x * kPlanThreads + tid; slot < total_up;
       slot += gridDim.x * kPlanThreads) {
    int lo = 0, hi = g_total - 1;  // last group with base <= slot
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_gbase[mid] <= slot) lo = mid; else hi = mid - 1;
    }
    int o0, o1;
    group_range(lo, o0, o1);
    const int rel = slot - s_gbase[lo];
    int i, o;
    if (merge && lo == 0) {
      // row pair q holds predicted tiles (2q, 2q+1) of each of the sz0 predicted blocks,
      // then the dense tile pairs p in [ceil(q Dp / Q), ceil((q+1) Dp / Q)) of each dense
      // block; row q starts at 2 q sz0 + 2 n_dense ceil(q Dp / Q)
      const int Q = s_q, Dp = s_dp;
      auto pfirst = [&](int q) { return (q * Dp + Q - 1) / Q; };
      auto base = [&](int q) { return 2 * q * sz0 + 2 * n_dense * pfirst(q); };
      int ql = 0, qh = Q - 1;
      while (ql < qh) {
        const int mid = (ql + qh + 1) >> 1;
        if (base(mid) <= rel) ql = mid; else qh = mid - 1;
      }
      const int q = ql, r2 = rel - base(q);
      if (r2 < 2 * sz0) {
        const int h = r2 & 1;
        o = n_dense + (r2 >> 1);
        i = 2 * q + h;
        if (h == 1 && i == s_nup[o]) i -= 1;
      } else {
        const int r3 = r2 - 2 * sz0, h = r3 & 1, c = pfirst(q + 1) - pfirst(q);
        const int dp = r3 >> 1;
        o = dp / c;                       // dense block (order)
        i = 2 * (pfirst(q) + dp % c) + h;
        if (i >= s_dn) i = s_dn - 1;      // odd tile count: repeat the last tile
      }
    } else if (a.pair_up) {
      // consecutive slots (2m, 2m + 1) = neuron tiles (2 i2, 2 i2 + 1) of ONE block: the
      // CTA pair running them shares the block's X tile by TMA multicast.  An odd tile
      // count repeats the block's last tile in the second slot (identical H writes).
      const int sz = o1 - o0;
      const int mx = (s_gbase[lo + 1] - s_gbase[lo]) / sz;  // tiles per block in this group
      const int pi = rel >> 1, h = rel & 1;
      int i2 = pi / sz;
      o = o0 + pi % sz;
      if (a.serpentine && (lo & 1)) i2 = mx / 2 - 1 - i2;
      i = 2 * i2 + h;
      if (h == 1 && i == s_nup[o]) i -= 1;
    } else {
      const int sz = o1 - o0;
      const int mx = (s_gbase[lo + 1] - s_gbase[lo]) / sz;
      i = rel / sz;
      o = o0 + rel % sz;
      // serpentine: odd groups sweep the neuron tiles downwards, so the weight rows the
      // previous group touched last are still in L2 when the next group starts
      if (a.serpentine && (lo & 1)) i = mx - 1 - i;
    }
    Tile t{-1, 0, 0, 0};
    if (i < s_ngu[o]) {
      t = Tile{order_to_block(o, a), i * 128, 0, 0};
    } else if (i < s_nup[o]) {
      t = Tile{order_to_block(o, a), (i - s_ngu[o]) * kUpBN, 1, 0};
    }
    up[slot] = t;
  }

  // down projection: groups of down_group blocks (raster order), column-tile major.
  // Paired (pair_down): slots (2m, 2m + 1) = column tiles (2 j2, 2 j2 + 1) of one block,
  // sharing its H tile by multicast; an odd column count pads the pair with a shadow
  // tile (kind 3: same tile, epilogue stores skipped -- the residual add is in place).
  const int nt = a.d / a.bn_down;
  const int ntp = a.pair_down ? rup(nt, 2) : nt;
  const int total_down = min(a.n_blk * ntp, down_cap);
  for (int slot = blockIdx.x * kPlanThreads + tid; slot < total_down;
       slot += gridDim.x * kPlanThreads) {
    const int g = slot / (a.down_group * ntp);
    const int o0 = g * a.down_group;
    const int sz = min(a.down_group, a.n_blk - o0);
    const int rel = slot - o0 * ntp;
    int j, o, kind = 2;
    if (a.pair_down) {
      const int pi = rel >> 1, h = rel & 1;
      j = 2 * (pi / sz) + h;
      o = o0 + pi % sz;
      if (j == nt) {
        j = nt - 1;
        kind = 3;
      }
    } else {
      j = rel / sz;
      o = o0 + rel % sz;
    }
    down[slot] = Tile{order_to_block(o, a), j * a.bn_down, kind,
                      (a.serpentine && (g & 1)) ? 1 : 0};
  }
  if (blockIdx.x == 0 && tid == 0) {
    pc->n_up = total_up;
    pc->n_down = total_down;
    pc->hcols = s_hcols;
    pc->next_down = 0;
    pc->next_up = 0;
  }
  if (!a.counts && FFWD_PLAN_BESIDE_TOPK) pdl_wait();
}

}  // namespace

cudaError_t launch_plan(const PlanArgs& a, BlockMeta* meta, Tile* up_tiles, int up_cap,
                        Tile* down_tiles, int down_cap, PlanCounts* counts, cudaStream_t s) {
  if (a.n_blk > kMaxBlocks) return cudaErrorInvalidValue;
  // every CTA rebuilds the per-block prefix (cheap) and writes its share of the slots
  const int ctas = (up_cap + down_cap + 4 * kPlanThreads - 1) / (4 * kPlanThreads);
  return launch_k(plan_kernel, dim3(ctas < 1 ? 1 : (ctas > 32 ? 32 : ctas)), dim3(kPlanThreads), 0,
                  s, 1, a, meta, up_tiles, up_cap, down_tiles, down_cap, counts);
}

}  // namespace ffwd
