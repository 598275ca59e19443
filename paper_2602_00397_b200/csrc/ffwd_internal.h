// Internal launch interfaces shared by the kernel translation units and the
// C-ABI shim (capi.cu).  Not part of the public boundary (include/ffwd_b200.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace ffwd {

constexpr int kBlockTokens = 128;  // model.py:25 block_size; one UMMA M tile

// Per-block metadata written by the plan kernel (one int4 pair per block).
struct BlockMeta {
  int tok0;      // first token row of the block in X / Y
  int ntok;      // tokens in the block (<= 128; short tail block)
  int kcount;    // neurons contracted: k_b (sparse) or f_local (dense)
  int kpad;      // kcount rounded up to 64 (H columns of the FFN part)
  int comp;      // compensator columns in H (rc rounded to 64) or 0
  int idx_row;   // row of the index buffer, -1 = identity (dense block)
  int ktot;      // kpad + comp : K extent of the down projection
  int n_gu;      // gate/up tiles (128 neurons each) for the up projection
  int n_up;      // up-projection slots of the block (incl. a pair's repeated tile)
};

// Tile table entry: block id + packed (kind, offset).  b < 0 = empty slot.
struct Tile {
  int b;
  int n0;    // neuron position (gate/up), comp column (comp) or output column (down)
  int kind;  // 0 = gate/up, 1 = compensator hidden, 2 = down, 3 = down shadow (no stores)
  int pad;   // down tiles: 1 = walk the K stages from the top down (serpentine raster)
};

struct PlanCounts {
  int n_up;       // entries in the up-projection tile table
  int n_down;     // entries in the down-projection tile table
  int hcols;      // H row stride actually used (<= the allocated stride)
  int next_down;  // dynamic tile claiming of the down projection (zeroed by the plan)
  int next_up;    // ... of the up projection (in CTA-pair units when paired)
  int pad[3];
};

// ------------------------------------------------------------------ K1
// Attention pooling: per-token logits (skipped with `logits_in`), a per-block softmax
// (`probs`: blk_count * 128 floats), the pooled sum; then the two f64-accumulated
// predictor GEMMs (DMMA, split-K partials reduced in fixed order).  `logits`:
// blk_count * 128 floats of scratch.
cudaError_t launch_pool(const void* x, bool x_is_f32, int T, int d, int blk_begin,
                        int blk_count, const float* query, float sqrt_d, float* logits,
                        float* pooled, const float* logits_in, float* probs, cudaStream_t s);
// Any-shape pooling: blocks of `rpb` rows, any d (the drop-in's small shapes).
cudaError_t launch_pool_generic(const void* x, bool x_is_f32, int T, int d, int rpb,
                                int blk_begin, int blk_count, const float* query, float sqrt_d,
                                float* pooled, cudaStream_t s);
// First pass alone: logits[t] for rows [tok0, tok0 + ntok) of x.
cudaError_t launch_logits_only(const void* x, bool x_is_f32, int d, int tok0, int ntok,
                               const float* query, float sqrt_d, float* logits, cudaStream_t s);
// FFN-input producers of the full prefill (norm.cu).
cudaError_t launch_rmsnorm(float* x, const float* gain, int T, int d, double eps,
                           const void* add, int add_kind, void* out_bf16, float* out_f32,
                           const float* query, float sqrt_d, float* logits, int logit_row0,
                           int logit_row1, bool logits_from_f32, cudaStream_t s);
// Deadline of the cross-GPU spin waits (ffwd_set_spin_timeout_ms; default 60 s).
unsigned long long spin_timeout_ns();
// Fused tensor-parallel completion (allreduce.cu): out_p = residual + sum_q partial_q on
// every rank p (peer pointers), optional bf16 copy; flags: per-rank [2n + 1] words.
cudaError_t launch_allreduce_residual(const float* const* partial, float* const* out,
                                      void* const* xnext, unsigned* const* flags, int n,
                                      int rank, const float* residual, int T, int d,
                                      unsigned epoch, int max_ctas, cudaStream_t s);
// The same completion overlapped with the down projection: block by block (in the plan's
// raster order) once every rank's K3 has published all of the block's column tiles
// (ydone[p][b] reaching `target`, a running count).
cudaError_t launch_allreduce_overlap(const float* const* partial, float* const* out,
                                     void* const* xnext, unsigned* const* flags,
                                     const unsigned* const* ydone, int n, int rank,
                                     const float* residual, int T, int d, unsigned epoch,
                                     unsigned target, int sparse_begin, int sparse_count,
                                     int max_ctas, cudaStream_t s);
// sparse.hidden_column_scores over H [T x ld] (bf16 or f32) in blocks of `rpb` rows ->
// scores [ceil(T / rpb) x f]
cudaError_t launch_hidden_scores(const void* h, bool is_f32, int ld, int T, int f, int rpb,
                                 float* scores, cudaStream_t s);
cudaError_t launch_rope(void* qk, bool is_f32, int T, int row_stride, int k_col, int n_heads,
                        int d_head, const double* cos_t, const double* sin_t, const float* cos32,
                        const float* sin32, int pos0, cudaStream_t s);
// `partial` (nullable, gemm_f64acc_partial_bytes) enables split-K for long K.
size_t gemm_f64acc_partial_bytes(int M, int K, int N);
int gemm_f64acc_kernels(int M, int K, int N, bool has_partial);  // launches per call
cudaError_t launch_gemm_f64acc(const float* A, const float* B, float* C, int M, int K, int N,
                               bool relu, double* partial, cudaStream_t s);
// `mask` (nullable): also the selection bitmask of each row (ld_mask 32-bit words per row)
cudaError_t launch_topk(const float* scores, int n_rows, int f, int k, int tp_rank, int tp_size,
                        int32_t* idx_global, int ld_global, int32_t* idx_local, int ld_local,
                        int32_t* counts, cudaStream_t s, uint32_t* mask = nullptr,
                        int ld_mask = 0);
// rank tp_rank's local neuron lists + counts from selection bitmasks (rows of ld_mask words)
cudaError_t launch_mask_to_local(const uint32_t* mask, int ld_mask, int n_rows, int f_global,
                                 int tp_rank, int tp_size, int32_t* idx_local, int ld_local,
                                 int32_t* counts, cudaStream_t s);

// ------------------------------------------------------------------ K2/K3
struct PlanArgs {
  int T, d, f_local, rc_local;
  int n_blk;
  int sparse_begin, sparse_count;  // contiguous range of predicted blocks
  int k_shared;                    // k for sparse blocks when counts == nullptr
  const int32_t* counts;           // per sparse row counts (TP local) or nullptr
  int idx_shared;                  // all sparse blocks use index row 0
  int has_comp;
  int up_group;                    // blocks per raster group (up projection)
  int down_group;                  // blocks per raster group (down projection)
  int bn_down;                     // output columns per down tile
  int hcols_alloc;
  int serpentine;                  // odd up-projection raster groups sweep tiles downwards
  int pair_up;                     // up tiles ordered in (i, i+1) pairs of one block
  int pair_down;                   // down tiles ordered in (j, j+1) column pairs of one block
  int* blk_done;                   // nullable: per-block up-tile counters, zeroed here
};

cudaError_t launch_plan(const PlanArgs& a, BlockMeta* meta, Tile* up_tiles, int up_cap,
                        Tile* down_tiles, int down_cap, PlanCounts* counts, cudaStream_t s);

struct GemmArgs {
  const void* x;        // bf16 [T x d]
  const void* wgu_t;    // bf16 [(2 f_local + rc_rows) x d]  gate^T | up^T | Wc1^T
  int wgu_rows;
  const void* wd;       // bf16 [(f_local + rc_rows) x d]    W_down | Wc2
  int wd_rows;
  void* h;              // bf16 [n_blk*128 x hcols]
  int hcols;
  float* y;             // f32 [T x d]
  const float* residual;  // nullable: y = residual + FFN (may alias y; engine.py:308)
  void* x_next;         // nullable: bf16 copy of y for the next layer's input
  int T, d, f_local, n_blk;
  const int32_t* idx;   // local neuron ids, row stride ld_idx
  int ld_idx;
  const BlockMeta* meta;
  const Tile* up_tiles;
  int up_cap;
  const Tile* down_tiles;
  int down_cap;
  PlanCounts* counts;   // tile counts (read) and the dynamic-claim counters (atomics)
  int num_sms;
  int bn_down;
  int* blk_done;  // nullable: block-granular K2 -> K3 dependency (per-block done tiles)
  unsigned* y_done;  // nullable: per-block finished down tiles, released at system scope
                     // (the overlapped TP completion consumes blocks as they finish)
};

cudaError_t launch_up_proj(const GemmArgs& a, cudaStream_t s);
bool up_proj_paired();    // the up projection runs as CTA pairs (tile table in pairs)
bool down_proj_paired();  // the down projection runs as CTA pairs
cudaError_t launch_down_proj(const GemmArgs& a, cudaStream_t s);

// tensor-map encoder (driver entry point resolved once through the runtime)
CUresult encode_tmap_2d_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                             uint32_t box_inner, uint32_t box_rows);
CUresult encode_tmap_2d_bf16_sw(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                                uint32_t box_inner, uint32_t box_rows, bool swizzle128);

}  // namespace ffwd
