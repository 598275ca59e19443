// Microbenchmark: TMA 2-D tile loads vs tile::gather4 into shared memory (no MMA).
// Measures L2->SMEM delivery rate per SM for the access patterns of the up/down
// gather-GEMMs.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I../paper_2602_00397_b200/csrc tma_bench.cu -o tma_bench
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "sm100.cuh"

using namespace ffwd;

constexpr int kMaxStages = 4;
constexpr int kStageBytes = 32768;

struct Bars {
  uint64_t full[kMaxStages];
};

// mode 0: one 2-D tile (64 x 256 rows) per stage; mode 1: 64 gather4 (256 rows) per
// stage issued by one thread; mode 2: 64 gather4 issued by 4 warps (16 each).
__global__ void __launch_bounds__(512, 1)
    tma_kernel(const __grid_constant__ CUtensorMap tm_tile, const __grid_constant__ CUtensorMap tm_g,
               const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_a2,
               const __grid_constant__ CUtensorMap tm_g2, const int* __restrict__ rows_all, int n_rowsets, int iters, int stages, int mode,
               int kdim, unsigned long long* cycles, const __nv_bfloat16* wptr, int share_a) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(base + kMaxStages * kStageBytes + 1024 + kMaxStages * 16384);
  __shared__ int srows[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // barrier arrivals per fill: TMA modes count issuing warps; cp.async modes count threads
  const int nwarps_issue = (mode == 13 || mode == 14 || mode == 15) ? 16 : mode == 12 ? 8 : mode == 10 ? 8 : mode == 11 ? 16 : mode == 7 ? 128 : mode == 8 ? 256 : mode == 9 ? 128 + 2 :
                           mode == 5 ? 8 : (mode == 6 ? 16 : (mode >= 2 ? 4 : 1));
  if (threadIdx.x == 0) {
    for (int i = 0; i < kMaxStages; ++i) mbar_init(&bars->full[i], nwarps_issue);
    fence_barrier_init();
  }
  __syncthreads();
  const int* rows = rows_all + (blockIdx.x % n_rowsets) * 256;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) srows[i] = rows[i];
  __syncthreads();
  const uint64_t pol = policy_evict_normal();
  unsigned long long t0 = clock64();
  uint32_t phase_bits = 0;
  const int nk = kdim / 64;
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    if (it >= stages) {  // wait for the stage's previous fill
      if (threadIdx.x == 0 || (mode == 2 && lane == 0 && warp < 4)) {
      }
      mbar_wait_sleep(&bars->full[s], (phase_bits >> s) & 1, 2000);
      phase_bits ^= 1u << s;
    }
    __syncthreads();
    const int kb = (it + (share_a > 1 ? blockIdx.x / share_a : blockIdx.x)) % nk;
    uint8_t* dst = base + s * kStageBytes;
    if (mode == 0) {
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes);
        tma_load_2d(&tm_tile, &bars->full[s], dst, kb * 64, (blockIdx.x * 256) % 16384, pol);
      }
    } else if (mode == 1) {
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes);
        const int4* rq = reinterpret_cast<const int4*>(srows);
        for (int q = 0; q < 64; ++q) {
          const int4 r = rq[q];
          tma_gather4(&tm_g, &bars->full[s], dst + q * 512, kb * 64, r.x, r.y, r.z, r.w, pol);
        }
      }
    } else if (mode == 2) {
      if (warp < 4 && lane == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes / 4);
        const int4* rq = reinterpret_cast<const int4*>(srows) + warp * 16;
        for (int q = 0; q < 16; ++q) {
          const int4 r = rq[q];
          tma_gather4(&tm_g, &bars->full[s], dst + (warp * 16 + q) * 512, kb * 64, r.x, r.y, r.z,
                      r.w, pol);
        }
      }
    } else if (mode == 3) {  // 4 warps, rows preloaded, fully unrolled issue
      if (warp < 4 && lane == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes / 4);
        const int4* rq = reinterpret_cast<const int4*>(srows) + warp * 16;
        int4 r[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) r[q] = rq[q];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          tma_gather4(&tm_g, &bars->full[s], dst + (warp * 16 + q) * 512, kb * 64, r[q].x,
                      r[q].y, r[q].z, r[q].w, pol);
      }
    } else if (mode == 12) {
      uint32_t cs, crank;
      asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
      asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
      if (warp < 8 && lane == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes / 8 + (warp == 0 ? 16384 : 0));
        if (warp == 0) {
          const uint32_t rows_each = 128 / cs;
          uint8_t* adst = base + kMaxStages * kStageBytes + 1024 + s * 16384 + crank * rows_each * 128;
          const uint16_t mask = (1u << cs) - 1;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(adst)),
              "l"(reinterpret_cast<uint64_t>(&tm_a2)), "r"(smem_u32(&bars->full[s])), "r"(kb * 64),
              "r"(int(((blockIdx.x / cs) * 128 + crank * rows_each) % 16384)), "h"(mask)
              : "memory");
        }
        const int4* rq = reinterpret_cast<const int4*>(srows) + warp * 8;
        for (int q = 0; q < 8; ++q) {
          const int4 r = rq[q];
          tma_gather4(&tm_g, &bars->full[s], dst + (warp * 8 + q) * 512, kb * 64, r.x, r.y, r.z,
                      r.w, pol);
        }
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 15) {
      // mode 14's pattern (64 rows x 4 chunks per stage) from a CHUNK-MAJOR copy of the
      // matrix ([kdim/64][rows][64]): the 4 chunks of a row are 2 MiB apart, not adjacent
      const int per = 16 / 16;
      const int kb2 = (it + blockIdx.x) % (kdim / 256);
      if (warp < 16 && lane == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes / 16);
        const int4* rq = reinterpret_cast<const int4*>(srows) + warp * per;
        for (int q = 0; q < per; ++q) {
          const int4 r = rq[q];
          for (int c = 0; c < 4; ++c) {
            const int cr = (kb2 * 4 + c) * 16384;
            tma_gather4(&tm_g2, &bars->full[s], dst + ((warp * per + q) * 4 + c) * 512, 0,
                        cr + r.x, cr + r.y, cr + r.z, cr + r.w, pol);
          }
        }
      }
    } else if (mode == 13 || mode == 14) {
      // 16 warps, same 32 KiB per stage, but each 4-row group fetches `nch` ADJACENT
      // 128 B column chunks back to back (mode 13: 128 rows x 2 chunks, the interleaved
      // gate/up layout; mode 14: 64 rows x 4 chunks, the down-projection pattern).
      const int nch = mode == 13 ? 2 : 4, groups = 64 / nch, per = groups / 16;
      const int kb2 = (it + blockIdx.x) % (kdim / (64 * nch));
      if (warp < 16 && lane == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes / 16);
        const int4* rq = reinterpret_cast<const int4*>(srows) + warp * per;
        for (int q = 0; q < per; ++q) {
          const int4 r = rq[q];
          for (int c = 0; c < nch; ++c)
            tma_gather4(&tm_g, &bars->full[s], dst + ((warp * per + q) * nch + c) * 512,
                        (kb2 * nch + c) * 64, r.x, r.y, r.z, r.w, pol);
        }
      }
    } else if (mode >= 10) {  // K2-like stage: 32 KiB gathered + 16 KiB A tile
      const int nw = mode == 10 ? 8 : 16, per = 64 / nw;
      if (warp < nw && lane == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes / nw + (warp == 0 ? 16384 : 0));
        if (warp == 0)
          tma_load_2d(&tm_a, &bars->full[s], base + kMaxStages * kStageBytes + 1024 + s * 16384,
                      kb * 64, ((share_a > 1 ? blockIdx.x / share_a : blockIdx.x) * 128) % 16384, pol);
        const int4* rq = reinterpret_cast<const int4*>(srows) + warp * per;
        for (int q = 0; q < per; ++q) {
          const int4 r = rq[q];
          tma_gather4(&tm_g, &bars->full[s], dst + (warp * per + q) * 512, kb * 64, r.x, r.y,
                      r.z, r.w, pol);
        }
      }
    } else if (mode >= 7) {  // cp.async 16 B per thread (LDGSTS), swizzled like TMA
      const int nthr = mode == 7 ? 128 : (mode == 8 ? 256 : 128);
      const int rows_cp = mode == 9 ? 128 : 256;  // mode 9: half the rows via cp.async
      const int row0 = mode == 9 ? 128 : 0;
      if (mode == 9 && (warp == 4 || warp == 5) && lane == 0) {  // 2 warps: 32 gather4
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes / 4);
        const int4* rq = reinterpret_cast<const int4*>(srows) + (warp - 4) * 16;
        for (int q = 0; q < 16; ++q) {
          const int4 r = rq[q];
          tma_gather4(&tm_g, &bars->full[s], dst + ((warp - 4) * 16 + q) * 512, kb * 64, r.x,
                      r.y, r.z, r.w, pol);
        }
      }
      if (threadIdx.x < nthr) {
        const int c = threadIdx.x & 7;
        for (int rr = threadIdx.x >> 3; rr < rows_cp; rr += nthr >> 3) {
          const int row = row0 + rr;
          const __nv_bfloat16* src = wptr + static_cast<size_t>(srows[row]) * kdim + kb * 64 + c * 8;
          const uint32_t d = smem_u32(dst + row * 128 + ((c ^ (row & 7)) << 4));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars->full[s])) : "memory");
      }
    } else if (mode >= 5) {  // 8 or 16 issuing warps
      const int nw = mode == 5 ? 8 : 16, per = 64 / nw;
      if (warp < nw && lane == 0) {
        mbar_arrive_expect_tx(&bars->full[s], kStageBytes / nw);
        const int4* rq = reinterpret_cast<const int4*>(srows) + warp * per;
        for (int q = 0; q < per; ++q) {
          const int4 r = rq[q];
          tma_gather4(&tm_g, &bars->full[s], dst + (warp * per + q) * 512, kb * 64, r.x, r.y,
                      r.z, r.w, pol);
        }
      }
    } else {  // mode 4: all 4 warps, each lane issues 0.5 gather4 (lanes 0..15), waterfall
      if (warp < 4) {
        if (lane == 0) mbar_arrive_expect_tx(&bars->full[s], kStageBytes / 4);
        __syncwarp();
        if (lane < 16) {
          const int4 r = reinterpret_cast<const int4*>(srows)[warp * 16 + lane];
          tma_gather4(&tm_g, &bars->full[s], dst + (warp * 16 + lane) * 512, kb * 64, r.x, r.y,
                      r.z, r.w, pol);
        }
      }
    }
  }
  // drain
  for (int i = 0; i < stages && i < iters; ++i) {
    const int it = iters - stages + i;
    if (it < 0) continue;
    const int s = it % stages;
    mbar_wait_sleep(&bars->full[s], (phase_bits >> s) & 1, 2000);
    phase_bits ^= 1u << s;
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int rows_total = 16384, kdim = 4096;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  void* w;
  cudaMalloc(&w, size_t(rows_total) * kdim * 2);
  cudaMemset(w, 0, size_t(rows_total) * kdim * 2);
  CUtensorMap tile, g;
  cuuint64_t dims[2] = {cuuint64_t(kdim), cuuint64_t(rows_total)};
  cuuint64_t str[1] = {cuuint64_t(kdim) * 2};
  cuuint32_t box_t[2] = {64, 256}, box_g[2] = {64, 1}, es[2] = {1, 1};
  enc(&tile, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box_t, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap amap;
  cuuint32_t box_a[2] = {64, 128};
  enc(&amap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box_a, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int promo = argc > 2 ? atoi(argv[2]) : 3;
  const int share = argc > 3 ? atoi(argv[3]) : 1;  // CTAs sharing one A tile stream
  const int csz = argc > 4 ? atoi(argv[4]) : 2;     // cluster size for mode 12
  CUtensorMap amap2;
  cuuint32_t box_a2[2] = {64, cuuint32_t(128 / csz)};
  enc(&amap2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box_a2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("A shared by %d CTAs\n", share);  // 0 none, 1 64B, 2 128B, 3 256B
  enc(&g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box_g, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("gather promotion %d\n", promo);
  CUtensorMap g2;  // chunk-major view: [kdim/64 * rows_total] rows of 64 elements
  cuuint64_t dims2[2] = {64, cuuint64_t(rows_total) * (kdim / 64)};
  cuuint64_t str2[1] = {128};
  enc(&g2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims2, str2, box_g, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)promo,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int n_sets = 148;
  std::vector<int> hrows(n_sets * 256);
  srand(1);
  const int span = argc > 1 ? atoi(argv[1]) : 2048;  // row window the gathered rows come from
  for (int s = 0; s < n_sets; ++s) {
    int lo = span < rows_total ? (s * 97) % (rows_total - span) : 0;
    std::vector<int> pick;
    for (int i = 0; i < 256; ++i) pick.push_back(lo + (rand() % span));
    std::sort(pick.begin(), pick.end());
    for (int i = 0; i < 256; ++i) hrows[s * 256 + i] = pick[i];
  }
  int* drows;
  cudaMalloc(&drows, hrows.size() * 4);
  cudaMemcpy(drows, hrows.data(), hrows.size() * 4, cudaMemcpyHostToDevice);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, 148 * 8);
  const size_t smem = 1024 + kMaxStages * kStageBytes + 1024 + kMaxStages * 16384 + sizeof(Bars);
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  const char* names[16] = {"tile 64x256", "gather4 x64 (1 thread)", "gather4 x64 (4 warps)",
                          "gather4 4w preload", "gather4 4w x16 lanes", "gather4 8 warps",
                          "gather4 16 warps", "cp.async 128 thr", "cp.async 256 thr",
                          "half gather4 + half cp.async", "K2 stage, 8 warps", "K2 stage, 16 warps", "K2 stage 8w A-multicast", "gather4 16w 2 adjacent chunks", "gather4 16w 4 adjacent chunks", "gather4 16w 4 chunks, chunk-major"};
  for (int mode = 0; mode < 16; ++mode) {
    if (mode == 1 || mode == 3 || mode == 4 || mode == 7 || mode == 9) continue;
    for (int stages : {4}) {
      if (mode != 12) tma_kernel<<<148, 512, smem>>>(tile, g, amap, amap2, g2, drows, n_sets, 50, stages, mode, kdim, dcyc, (const __nv_bfloat16*)w, share);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (mode == 12) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, tma_kernel, tile, g, amap, amap2, g2, (const int*)drows, n_sets, iters,
                           stages, mode, kdim, dcyc, (const __nv_bfloat16*)w, share);
      } else
      tma_kernel<<<148, 512, smem>>>(tile, g, amap, amap2, g2, drows, n_sets, iters, stages, mode, kdim, dcyc, (const __nv_bfloat16*)w, share);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> c(148);
      cudaMemcpy(c.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto v : c) avg += v;
      avg /= 148;
      const double bytes = 148.0 * iters * (kStageBytes + (mode >= 10 && mode <= 12 ? 16384 : 0));
      printf("%-24s stages=%d span=%d: %.1f cyc/stage/SM, %.2f TB/s aggregate (%.3f ms) %s\n",
             names[mode], stages, span, avg / iters, bytes / (ms * 1e-3) / 1e12, ms,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
