/*
 * ffwd_b200.h — C-ABI boundary of the B200-native FastForward prefill-FFN hot path.
 *
 * The reference (arXiv 2602.00397, /root/reference/pkg/src/sparseprefill) has no
 * FFI: the path is plain Python calls from engine.py:284-300.  These entry points
 * are what a binding of that path needs; each one names the
 * reference function(s) it replaces.  The Python package
 * paper_2602_00397_b200 binds them with ctypes.
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *     buffers are caller owned and never retained after return;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); all work is
 *     stream ordered, nothing synchronises the host;
 *   - bf16 buffers are passed as `const void*` (IEEE bfloat16, row-major);
 *   - return value: FFWD_OK or an error code; ffwd_last_error() gives the
 *     message (thread local).  FFWD_ERR_VALIDATION mirrors the reference's
 *     ValidationError (errors.py:9) and is raised before any launch.
 *
 * Weight layouts (built once per layer by paper_2602_00397_b200.layer.pack_layer):
 *   wgu_t  bf16 [(2*f_local + rc_up_rows) x d]  rows: gate^T | up^T | Wc1^T | 0-pad
 *          (model.py:79 w_gate/w_up (d, f) transposed to neuron-major;
 *           compensator.py:25-39 w1 (d, r') transposed), rc_up_rows = roundup(rc_local, 256)
 *   wd     bf16 [(f_local + rc_dn_rows) x d]    rows: W_down | Wc2 | 0-pad,
 *          rc_dn_rows = roundup(rc_local, 64)
 *   Under tensor parallelism rank s holds neurons {j : j % tp_size == s} (local
 *   row j / tp_size) and compensator columns [s*rc/tp, (s+1)*rc/tp).
 */
#ifndef FFWD_B200_H
#define FFWD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FFWD_API __attribute__((visibility("default")))
#else
#define FFWD_API
#endif

#define FFWD_ABI_VERSION 1

#define FFWD_OK 0
#define FFWD_ERR_VALIDATION 1  /* bad shape / k / index set  -> ValidationError */
#define FFWD_ERR_CUDA 2        /* CUDA runtime or launch error -> RuntimeError  */
#define FFWD_ERR_UNSUPPORTED 3 /* no sm_100 device / shape outside kernel limits */

FFWD_API int ffwd_abi_version(void);
FFWD_API const char* ffwd_last_error(void);

/* 0 when `device` is an sm_100 (B200-class) GPU; FFWD_ERR_UNSUPPORTED otherwise. */
FFWD_API int ffwd_device_check(int device);

/* Tuning knobs of the gather-GEMM rasterisation (blocks per L2 group). */
FFWD_API int ffwd_set_raster(int up_group, int down_group);
/*
 * Deadline of the cross-GPU waits of the peer-memory completions (ffwd_allreduce_residual,
 * ffwd_ffn_layer_tp_overlap): a rank that waits longer than `ms` for a peer traps (the
 * CUDA context reports an error) instead of hanging the GPU.  Default 60000 ms, so
 * ordinary rank skew (first-iteration setup, a host-side pause) is waited out.
 */
FFWD_API int ffwd_set_spin_timeout_ms(int ms);

/* Tuning knob: odd up-projection raster groups sweep their neuron tiles downwards (1,
 * default) so the previous group's last weight rows are still in L2. */
FFWD_API int ffwd_set_serpentine(int on);
/* Programmatic dependent launch of the hot-path kernels (1, default): each kernel's
 * prologue overlaps its predecessor's tail; 0 = plain stream serialisation. */
FFWD_API int ffwd_set_pdl(int on);

/*
 * Predictor scores for blocks [blk_begin, blk_begin + blk_count) of x.
 * Replaces predictor.py:68-81 predictor_forward (called per block at engine.py:286):
 *   scores[i, :] = relu(f32(pool(x_blk) . w1)) . w2 with f64 accumulation,
 *   bit-identical to the reference.
 * x: [T x d] f32 (x_is_f32 = 1) or bf16; query f32 [d]; w1 f32 [d x r];
 * w2 f32 [r x f]; scores f32 [blk_count x f].
 */
FFWD_API size_t ffwd_predictor_workspace_bytes(int blk_count, int d, int r, int f);
FFWD_API int ffwd_predictor_forward(const void* x, int x_is_f32, int T, int d, int blk_begin,
                           int blk_count, const float* query, const float* w1, const float* w2,
                           int r, int f, float* scores, void* workspace,
                           size_t workspace_bytes, void* stream);

/*
 * predictor_forward (predictor.py:68-81) for ONE block of any n rows and any d_model:
 * the reference pools whatever block it is handed (n = 1 .. 25600 here), so the drop-in
 * accepts what it accepts.  x [n x d] (bf16, or f32 when x_is_f32); scores [f] f32;
 * workspace >= ffwd_predictor_workspace_bytes(1, d, r, f).  Same f64 accumulation and
 * f32 rounding points as ffwd_predictor_forward.
 */
FFWD_API int ffwd_predictor_forward_block(const void* x, int x_is_f32, int n, int d,
                                          const float* query, const float* w1, const float* w2,
                                          int r, int f, float* scores, void* workspace,
                                          size_t workspace_bytes, void* stream);

/*
 * The predictor's first pooling pass alone (predictor.py:76): logits[t] =
 * f32(q . x_t) / f32(sqrt d) for every row t of x [T x d] (bf16, or f32 when
 * x_is_f32), f64 accumulation in the fixed order the fused RMSNorm producer shares
 * (ffwd_rmsnorm_ex), so either source gives bit-identical logits.  d % 4 == 0.
 */
FFWD_API int ffwd_predictor_logits(const void* x, int x_is_f32, int T, int d, const float* query,
                                   float* logits, void* stream);

/*
 * Per-row top-k.  Replaces kernels.py:139-149 topk_indices / sparse.py:49-55 build_mask:
 * ties keep the lower index, -0 == +0, NaN after every number, result ascending.
 * idx_global [n_rows x ld_global] (nullable) receives global neuron ids; with
 * tp_size > 1, idx_local [n_rows x ld_local] (nullable) receives the rank-local
 * ids j / tp_size of the selected neurons with j % tp_size == tp_rank and
 * counts [n_rows] (nullable) their number.
 */
FFWD_API int ffwd_topk(const float* scores, int n_rows, int f, int k, int tp_rank, int tp_size,
              int32_t* idx_global, int ld_global, int32_t* idx_local, int ld_local,
              int32_t* counts, void* stream);

/* predictor_forward + build_mask fused into one stream-ordered call. */
FFWD_API int ffwd_predict_topk(const void* x, int x_is_f32, int T, int d, int blk_begin, int blk_count,
                      const float* query, const float* w1, const float* w2, int r, int f, int k,
                      int tp_rank, int tp_size, int32_t* idx_global, int ld_global,
                      int32_t* idx_local, int ld_local, int32_t* counts, void* workspace,
                      size_t workspace_bytes, void* stream);

/*
 * Sparse SwiGLU FFN (+ optional compensator) over every 128-token block of x.
 * Replaces sparse.py:66-91 select_subweights + sparse_ffn_forward and, with
 * has_comp, compensator.py:52-66 compensator_forward + apply_compensation; with
 * idx == NULL it is engine.py:127-131 dense_ffn.
 * idx: [n_idx_rows x ld_idx] int32 ascending rank-local neuron ids; one row per
 * block when idx_per_block, else row 0 is shared by all blocks; counts
 * (nullable) gives per-row k, else k for every row.
 * y: f32 [T x d] (partial sum of this rank under tensor parallelism).
 */
FFWD_API size_t ffwd_sparse_ffn_workspace_bytes(int T, int d, int f_local, int rc_local, int k);
FFWD_API int ffwd_sparse_ffn(const void* x_bf16, int T, int d, const void* wgu_t, const void* wd,
                    int f_local, int rc_local, const int32_t* idx, int idx_per_block, int ld_idx,
                    const int32_t* counts, int k, int has_comp, float* y, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * One layer of the FFN branch of the block-wise prefill, all blocks at once.
 * Replaces the engine.py:254-310 FFN branch (mode "predicted") for one layer:
 * dense first/last block when dense_first_last (engine.py:258-262; 1 = the whole
 * prompt, 2 / 3 = a sequence shard holding only the prompt's first / last block, so
 * only that one is dense; 0 = none), dense when
 * k >= f_global (engine.py:268), otherwise predictor -> top-k -> sparse FFN ->
 * compensation (has_comp).  The residual add (engine.py:308) stays with the
 * caller unless `residual` is given: then y = residual + FFN(x) (y may alias
 * residual), fused into the down-projection epilogue; x_next_bf16 (nullable)
 * receives bf16(y) as the next layer's input.  Both need tp_size == 1 (under
 * tensor parallelism the all-reduce comes first).  idx_global (nullable,
 * [n_sparse x ld_idx_global]) receives the selected global neuron ids of every
 * predicted block.
 */
FFWD_API size_t ffwd_layer_workspace_bytes(int T, int d, int f_global, int f_local, int rc_local, int r,
                                  int k, int dense_first_last, int tp_size);
FFWD_API int ffwd_ffn_layer(const void* x_bf16, int T, int d, const void* wgu_t, const void* wd,
                   int f_local, int rc_local, const float* query, const float* w1,
                   const float* w2, int r, int f_global, int k, int dense_first_last,
                   int has_comp, int tp_rank, int tp_size, float* y, const float* residual,
                   void* x_next_bf16, int32_t* idx_global, int ld_idx_global, void* workspace,
                   size_t workspace_bytes, void* stream);

/*
 * Oracle scoring (sparse.py:94-115 oracle_experts / hidden_column_scores): the
 * dense gate/up products of every 128-token block of x (identity index, no
 * compensator), H = silu(x Wg) * (x Wu) in bf16, then per block and neuron
 * scores[b][j] = f32(sqrt(sum_t H[t][j]^2)) (f64 sum).  tp_size 1 layout
 * (f = d_ffn rows of gate^T / up^T in wgu_t).  scores: f32 [n_blk x f].
 */
FFWD_API size_t ffwd_hidden_scores_workspace_bytes(int T, int d, int f);
FFWD_API int ffwd_hidden_scores(const void* x_bf16, int T, int d, const void* wgu_t, int f,
                                int rc_local, float* scores, void* workspace,
                                size_t workspace_bytes, void* stream);

/*
 * sparse.hidden_column_scores (sparse.py:94-97) of a hidden matrix h [n_rows x f]
 * (row stride ld; f32 when is_f32 else bf16), per 128-row block:
 * scores[b][j] = f32(sqrt(sum_t h[t][j]^2)), f64 sum.  scores: f32 [ceil(n/128) x f].
 */
FFWD_API int ffwd_column_norms(const void* h, int is_f32, int n_rows, int ld, int f,
                               float* scores, void* stream);

/*
 * The FFN branch of engine.py:254-310 for the ablation modes (tp_size 1):
 *   mode 1 "oracle": every sparse block is scored by its own dense gate/up pass
 *                    (oracle_experts) and keeps its top-k;
 *   mode 2 "static": block 0 runs dense and its hidden-norm top-k (mask_from_hidden,
 *                    FirstBlockStatic) is used by every later sparse block.
 * Dense blocks as in the engine (dense_first_last, static block 0, k >= f).
 * idx_out (nullable) receives the masks: [n_scored x ld_idx_out] (1 row for static).
 */
FFWD_API size_t ffwd_ffn_layer_mode_workspace_bytes(int T, int d, int f, int rc_local, int k,
                                                    int mode, int dense_first_last);
FFWD_API int ffwd_ffn_layer_mode(const void* x_bf16, int T, int d, const void* wgu_t,
                                 const void* wd, int f, int rc_local, int k, int mode,
                                 int dense_first_last, int has_comp, float* y,
                                 const float* residual, void* x_next_bf16, int32_t* idx_out,
                                 int ld_idx_out, void* workspace, size_t workspace_bytes,
                                 void* stream);

/*
 * ffwd_ffn_layer with two optional predictor inputs (NULL = as ffwd_ffn_layer):
 *   x_pred_f32  f32 [T x d]: the predictor pools over these values instead of
 *               x_bf16 -- the reference predictor sees the f32 RMSNorm output
 *               (engine.py:267, 285), so exact full-model parity uses it;
 *   logits_in   f32 [T]: per-token predictor logits f32(q . x_t) / f32(sqrt d)
 *               (predictor.py:76) already produced by the FFN-input producer
 *               (ffwd_rmsnorm with a query), which skips the pooling's first pass.
 */
FFWD_API int ffwd_ffn_layer2(const void* x_bf16, int T, int d, const void* wgu_t, const void* wd,
                    int f_local, int rc_local, const float* query, const float* w1,
                    const float* w2, int r, int f_global, int k, int dense_first_last,
                    int has_comp, int tp_rank, int tp_size, float* y, const float* residual,
                    void* x_next_bf16, int32_t* idx_global, int ld_idx_global,
                    const float* x_pred_f32, const float* logits_in, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * The sequence-parallel predictor (tp.SeqParallelTP): under tensor parallelism each rank
 * predicts only the blocks of its own T/N residual rows and the ranks all-gather the
 * selections as bitmasks, instead of every rank predicting every block.
 *
 * ffwd_predict_mask: predictor_forward + build_mask (predictor.py:68-81,
 * kernels.py:139-149, sparse.py:49-55) for blocks [blk_begin, blk_begin + blk_count) of
 * x [T x d] (bf16, or f32 when x_is_f32), with the per-token logits from the FFN-input
 * producer when logits_in (f32 [T]) is given.  Row i of `mask` (ld_mask >= ceil(f / 32)
 * 32-bit words per row) receives block blk_begin + i's selection: bit j of word j / 32 =
 * neuron j kept.  Bit-identical to the indices ffwd_ffn_layer2 selects for those blocks.
 */
FFWD_API size_t ffwd_predict_mask_workspace_bytes(int blk_count, int d, int r, int f);
FFWD_API int ffwd_predict_mask(const void* x, int x_is_f32, int T, int d, int blk_begin,
                               int blk_count, const float* query, const float* w1,
                               const float* w2, int r, int f, int k, const float* logits_in,
                               uint32_t* mask, int ld_mask, void* workspace,
                               size_t workspace_bytes, void* stream);
/*
 * ffwd_ffn_layer2 with the selection given: `mask` holds one row per block of x (row b =
 * block b; only the predicted blocks' rows are read), in the ffwd_predict_mask format.
 * The rank keeps its own strided neurons of each row (local ids j / tp_size, ascending)
 * and runs the gather-GEMMs and compensator exactly as ffwd_ffn_layer2.  Workspace: the
 * ffwd_layer_workspace_bytes size suffices.
 */
FFWD_API int ffwd_ffn_layer_masked(const void* x_bf16, int T, int d, const void* wgu_t,
                                   const void* wd, int f_local, int rc_local, int f_global,
                                   int k, int dense_first_last, int has_comp, int tp_rank,
                                   int tp_size, const uint32_t* mask, int ld_mask, float* y,
                                   const float* residual, void* x_next_bf16, void* workspace,
                                   size_t workspace_bytes, void* stream);

/*
 * kernels.rmsnorm (kernels.py:96-106) of the f32 residual stream x [T x d]:
 * out = f32(x / sqrt(mean_f64(x^2) + eps) * gain), evaluated in f64 like the
 * reference, written to out_bf16 (bf16 [T x d]) and/or out_f32.  With `add`
 * ([T x d], f32 when add_kind == 1, bf16 when 2) the residual add x += add
 * (engine.py:265, the attention output) runs first and x is updated in place.  With a
 * predictor `query` (f32 [d]) it also writes logits[t - logit_row0] =
 * f32(q . bf16(out_t)) / f32(sqrt d) for rows t in [logit_row0, logit_row1):
 * the FFN-input producer fused with the predictor's first pass (engine.py:267
 * followed by predictor.py:76).  d % 4 == 0, d <= 16384.
 */
FFWD_API int ffwd_rmsnorm(float* x, const float* gain, int T, int d, double eps,
                          const void* add, int add_kind, void* out_bf16, float* out_f32,
                          const float* query, float* logits, int logit_row0, int logit_row1,
                          void* stream);

/*
 * ffwd_rmsnorm with flags.  FFWD_NORM_LOGITS_F32: the logits are f32(q . out_f32_t) /
 * f32(sqrt d), i.e. dotted with the f32 output instead of its bf16 rounding (needs
 * out_f32); the predictor then pools that f32 copy (ffwd_ffn_layer2's x_pred_f32), as
 * the reference's predictor sees the f32 FFN input (engine.py:267, :286).  Either way
 * the f64 summation order is the one ffwd_predictor_forward's own first pass uses, so
 * the fused logits are bit-identical to the unfused ones.
 */
#define FFWD_NORM_LOGITS_F32 1
FFWD_API int ffwd_rmsnorm_ex(float* x, const float* gain, int T, int d, double eps,
                             const void* add, int add_kind, void* out_bf16, float* out_f32,
                             const float* query, float* logits, int logit_row0, int logit_row1,
                             int flags, void* stream);

/*
 * apply_rope (engine.py:50-68) in place on Q and K of one [T x row_stride]
 * buffer (bf16, or f32 when is_f32): Q heads at columns [0, n_heads*d_head),
 * K heads at [k_col, k_col + n_heads*d_head).  Token t sits at position
 * pos0 + t; cos_t / sin_t are f64 [max_pos x d_head/2] tables of
 * cos/sin(pos * 10000^(-2i/d_head)).  f32 storage is rotated in f64 (bit-exact to
 * the reference); bf16 storage in f32 from cos32 / sin32 (f32 copies of the tables;
 * NULL = the f64 path).
 */
FFWD_API int ffwd_rope(void* qk, int is_f32, int T, int row_stride, int k_col, int n_heads,
                       int d_head, const double* cos_t, const double* sin_t, const float* cos32,
                       const float* sin32, int pos0, void* stream);

/*
 * `.ffwd` checkpoint reader (checkpoint.py:1-22 layout, read_checkpoint :207-263):
 * memory-maps the file, validates the header and directory with the reference's
 * rules (FFWD_ERR_VALIDATION + ffwd_ckpt_last_error on failure) and exposes every
 * tensor as a zero-copy little-endian f32 host pointer into the mapping (valid
 * until ffwd_ckpt_close).  Host-only: no GPU needed.
 */
FFWD_API const char* ffwd_ckpt_last_error(void);
FFWD_API int ffwd_ckpt_open(const char* path, void** handle);
FFWD_API void ffwd_ckpt_close(void* handle);
FFWD_API const char* ffwd_ckpt_config(void* handle, size_t* len);
FFWD_API int ffwd_ckpt_num_tensors(void* handle);
FFWD_API int ffwd_ckpt_tensor(void* handle, int i, const char** name, int* ndim, uint32_t* dims,
                              const float** data, uint64_t* nbytes);

/*
 * Tensor-parallel completion of the down projection over NVLink peer memory, fused
 * with the residual add (engine.py:308): for this rank's row slice
 * [T*rank/n, T*(rank+1)/n) it reads every rank's partial Y from that rank's HBM,
 * adds the local residual rows and writes the result (and, if xnexts != NULL, its
 * bf16 copy) into every rank's output -- reduce-scatter + all-gather in one pass.
 * Host arrays of n device pointers (peer pointers from ffwd_ipc_open):
 *   partials[p]  f32 [T x d] rank p's partial Y (written by its down projection);
 *   outs[p]      f32 [T x d] rank p's residual stream (may alias its residual);
 *   xnexts[p]    bf16 [T x d] or NULL;
 *   flags[p]     u32 [2n + 1] zero-initialised sync words of rank p.
 * `epoch` must increase by one per call (flags are never reset).  Cross-GPU waits
 * are bounded and trap instead of hanging.  max_ctas <= 0: one CTA per SM (the grid
 * must be co-resident).
 */
FFWD_API int ffwd_allreduce_residual(const float* const* partials, float* const* outs,
                                     void* const* xnexts, unsigned* const* flags, int n_ranks,
                                     int rank, const float* residual, int T, int d,
                                     unsigned epoch, int max_ctas, void* stream);
/*
 * One tensor-parallel layer (as ffwd_ffn_layer2 with tp_size ranks) whose completion is
 * overlapped with the down projection: this rank's K3 writes its partial Y into
 * partials[tp_rank] and publishes, per 128-token block, how many column tiles are done
 * (y_done[tp_rank][b] += 1 per tile, system-scope release); a completion kernel on
 * `comm_stream` (comm_ctas CTAs, default 32) starts when this rank's up projection
 * retires and, block by block in the plan's raster order, waits for y_done[p][b] >=
 * y_epoch * (d / 256) on every rank p and then does ffwd_allreduce_residual's work for
 * its 1/N of the block's rows.  So the reduce-scatter + all-gather of block b over
 * NVLink runs while K3 still computes later blocks ("chunk over block
 * groups and overlap").  `stream` waits for the completion before returning work to the
 * caller.  y_done: caller-owned u32 [ceil(T/128)] per rank, zeroed once and never reset;
 * y_epoch counts the overlapped layers run on those counters (1, 2, ...); `epoch` is
 * ffwd_allreduce_residual's flag epoch.  xnexts must not alias x_bf16 (peers write the
 * next layer's input while this rank may still read this one).  Replaces
 * engine.py:294-308 (sparse FFN, compensator, residual) with the TP all-reduce of
 * SURVEY 8(e) fused in.
 */
FFWD_API int ffwd_ffn_layer_tp_overlap(const void* x_bf16, int T, int d, const void* wgu_t,
                                       const void* wd, int f_local, int rc_local,
                                       const float* query, const float* w1, const float* w2,
                                       int r, int f_global, int k, int dense_first_last,
                                       int has_comp, int tp_rank, int tp_size,
                                       int32_t* idx_global, int ld_idx_global,
                                       const float* x_pred_f32, const float* logits_in,
                                       const float* const* partials, float* const* outs,
                                       void* const* xnexts, unsigned* const* flags,
                                       unsigned* const* y_done, const float* residual,
                                       unsigned epoch, unsigned y_epoch, int comm_ctas,
                                       void* workspace, size_t workspace_bytes, void* stream,
                                       void* comm_stream);
/* CUDA IPC: the 64-byte handle of the allocation holding dev_ptr plus dev_ptr's
 * offset in it; ffwd_ipc_open maps a peer's allocation (add the offset). */
FFWD_API int ffwd_ipc_get_handle(void* dev_ptr, void* handle_out, size_t* offset_out);
FFWD_API int ffwd_ipc_open(const void* handle, void** dev_ptr);
FFWD_API int ffwd_ipc_close(void* dev_ptr);

/*
 * Per-launch device timing (CUDA events on the launching stream) for the
 * measurement harness.  Stages: 0 pool, 1 predictor W1, 2 predictor W2,
 * 3 top-k, 4 plan, 5 up-projection (K2), 6 down-projection (K3), 7 FFN-input
 * RMSNorm.  ffwd_timing_read waits for the recorded events, writes per-stage
 * summed milliseconds and kernel-launch counts, and clears the record.
 */
#define FFWD_N_STAGES 7
FFWD_API int ffwd_timing_enable(int on);
FFWD_API int ffwd_timing_read(double* ms_out, int* count_out, int n_stages);
FFWD_API const char* ffwd_stage_name(int stage);

#ifdef __cplusplus
}
#endif

#endif /* FFWD_B200_H */
