// extern "C" boundary (include/ffwd_b200.h): validation with the reference's
// error semantics, workspace carving, and the per-layer launch sequence
//   pool -> W1 -> W2 -> top-k -> plan -> up-proj (K2) -> down-proj (K3).
#include <cuda_bf16.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/ffwd_b200.h"
#include "ffwd_internal.h"

using namespace ffwd;

namespace {

thread_local std::string g_err;
// Process-wide tuning knobs: atomics, so a knob set from one thread is read whole by
// launches on any other (each launch reads each knob once; calls stay re-entrant).
std::atomic<int> g_up_group{32};
std::atomic<int> g_serpentine{1};
#ifndef FFWD_BLOCKDEP_DEFAULT
#define FFWD_BLOCKDEP_DEFAULT 1
#endif
std::atomic<int> g_blockdep{FFWD_BLOCKDEP_DEFAULT};
#ifndef FFWD_PDL_DEFAULT
#define FFWD_PDL_DEFAULT 1
#endif
std::atomic<int> g_pdl{FFWD_PDL_DEFAULT};
// ncu sweep: K3 DRAM 3.0 GB -> 1.7 GB per layer vs 8 (profiles/r1_raster_sweep.txt)
std::atomic<int> g_down_group{16};
std::atomic<long long> g_spin_timeout_ms{60000};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(FFWD_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define FFWD_CUDA(call, where)                    \
  do {                                            \
    cudaError_t _e = (call);                      \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

int rup(int v, int m) { return (v + m - 1) / m * m; }

// ---- optional per-launch event timing (measurement harness only)
enum Stage { kPool = 0, kW1, kW2, kTopk, kPlan, kUp, kDown, kNorm, kNumStages };
const char* kStageNames[kNumStages] = {"pool", "predictor_w1", "predictor_w2", "topk",
                                       "plan", "up_proj", "down_proj", "ffn_norm"};
std::atomic<bool> g_timing{false};
struct Rec {
  int stage;
  int kernels;  // kernel launches inside the timed stage
  cudaEvent_t a, b;
};
std::mutex g_rec_mu;  // guards g_recs and g_event_pool (launches may come from any thread)
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t take_event() {
  std::lock_guard<std::mutex> lk(g_rec_mu);
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct StageTimer {
  Rec r{-1, 1, nullptr, nullptr};
  cudaStream_t s;
  StageTimer(int stage, cudaStream_t st, int kernels = 1) : s(st) {
    if (!g_timing) return;
    r.stage = stage;
    r.kernels = kernels;
    r.a = take_event();
    r.b = take_event();
    cudaEventRecord(r.a, s);
  }
  ~StageTimer() {
    if (r.stage < 0) return;
    cudaEventRecord(r.b, s);
    std::lock_guard<std::mutex> lk(g_rec_mu);
    g_recs.push_back(r);
  }
};
size_t al(size_t v) { return (v + 255) & ~size_t(255); }

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

int bn_for(int d) { return d % 256 == 0 ? 256 : (d % 128 == 0 ? 128 : 64); }

// Workspace carve-out helper: sequential 256 B aligned sub-allocations.
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* p) : base(static_cast<char*>(p)) {}
  template <typename T>
  T* take(size_t n) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += al(n * sizeof(T));
    return p;
  }
};

struct Pred {
  float* logits;
  float* probs;  // f32(softmax) per block token (softmax_kernel)
  float* pooled;
  float* hidden;
  double* partial;
  float* scores;  // only carved when with_scores
};

Pred carve_pred(Carve& c, int nb, int d, int r, int f, bool with_scores) {
  Pred p;
  p.logits = c.take<float>(static_cast<size_t>(nb) * kBlockTokens);
  p.probs = c.take<float>(static_cast<size_t>(nb) * kBlockTokens);
  p.pooled = c.take<float>(static_cast<size_t>(nb) * d);
  p.hidden = c.take<float>(static_cast<size_t>(nb) * r);
  const size_t part = std::max(gemm_f64acc_partial_bytes(nb, d, r),
                               gemm_f64acc_partial_bytes(nb, r, f));
  p.partial = c.take<double>(part / sizeof(double));
  p.scores = with_scores ? c.take<float>(static_cast<size_t>(nb) * f) : nullptr;
  return p;
}

int run_predictor(const void* x, bool x_is_f32, int T, int d, int b0, int nb, const float* query,
                  const float* w1, const float* w2, int r, int f, const Pred& p, float* scores,
                  cudaStream_t s, const float* logits_in = nullptr) {
  const float sqrt_d = static_cast<float>(std::sqrt(static_cast<double>(d)));  // predictor.py:76
  if (d % 8 != 0) {  // any-shape pooling (small drop-in shapes; no fused logits)
    StageTimer tm(kPool, s);
    FFWD_CUDA(launch_pool_generic(x, x_is_f32, T, d, kBlockTokens, b0, nb, query, sqrt_d,
                                  p.pooled, s),
              "pool");
  } else {
    StageTimer tm(kPool, s, logits_in ? 2 : 3);  // [logits,] softmax, pool
    FFWD_CUDA(launch_pool(x, x_is_f32, T, d, b0, nb, query, sqrt_d, p.logits, p.pooled, logits_in,
                          p.probs, s),
              "pool");
  }
  {
    StageTimer tm(kW1, s, gemm_f64acc_kernels(nb, d, r, true));  // (the cluster path's count)
    FFWD_CUDA(launch_gemm_f64acc(p.pooled, w1, p.hidden, nb, d, r, true, p.partial, s), "w1");
  }
  {
    StageTimer tm(kW2, s);
    FFWD_CUDA(launch_gemm_f64acc(p.hidden, w2, scores, nb, r, f, false, nullptr, s), "w2");
  }
  return FFWD_OK;
}

struct Ffn {
  int32_t* idx_local;
  int32_t* counts;
  BlockMeta* meta;
  Tile* up;
  Tile* down;
  PlanCounts* pc;
  __nv_bfloat16* h;
  int* blk_done;
  int up_cap, down_cap, hcols, ld_local;
};

// kmax: largest per-block neuron count of a predicted block (rank local)
Ffn carve_ffn(Carve& c, int T, int d, int f_local, int rc_local, int kmax, int n_sparse,
              int ld_local) {
  Ffn w;
  const int n_blk = (T + kBlockTokens - 1) / kBlockTokens;
  const int rc64 = rup(rc_local, 64);
  const int tiles_dense = (f_local + 127) / 128;
  const int tiles_sparse = (kmax + 127) / 128 + (rc64 + 255) / 256;
  w.up_cap = n_blk * rup(tiles_dense > tiles_sparse ? tiles_dense : tiles_sparse, 2);
  w.down_cap = n_blk * rup(d / bn_for(d), 2);
  w.hcols = rup(rup(f_local, 64) > rup(kmax, 64) + rc64 ? rup(f_local, 64) : rup(kmax, 64) + rc64,
                64);
  w.ld_local = ld_local;
  w.idx_local = c.take<int32_t>(static_cast<size_t>(n_sparse > 0 ? n_sparse : 1) * ld_local);
  w.counts = c.take<int32_t>(n_sparse > 0 ? n_sparse : 1);
  w.meta = c.take<BlockMeta>(n_blk);
  w.up = c.take<Tile>(w.up_cap);
  w.down = c.take<Tile>(w.down_cap);
  w.pc = c.take<PlanCounts>(1);
  w.blk_done = c.take<int>(n_blk);
  w.h = c.take<__nv_bfloat16>(static_cast<size_t>(n_blk) * kBlockTokens * w.hcols);
  return w;
}

Ffn carve_ffn_at(void* ws, int T, int d, int f_local, int rc_local, int k) {
  Carve c(ws);
  return carve_ffn(c, T, d, f_local, rc_local, k, 0, 4);
}

int check_common(int T, int d, int f, int k) {
  if (T < 1) return fail(FFWD_ERR_VALIDATION, "token count must be >= 1, got %d", T);
  if (d < 1 || f < 1) return fail(FFWD_ERR_VALIDATION, "bad dims d=%d f=%d", d, f);
  if (k < 1 || k > f) return fail(FFWD_ERR_VALIDATION, "k=%d out of range [1, %d]", k, f);
  return FFWD_OK;
}

int run_ffn(const void* x, int T, int d, const void* wgu_t, const void* wd, int f_local,
            int rc_local, const Ffn& w, const int32_t* idx, int ld_idx, int sparse_begin,
            int sparse_count, const int32_t* counts, int k_shared, int idx_shared, int has_comp,
            float* y, const float* residual, void* x_next, cudaStream_t s,
            bool up_only = false, unsigned* y_done = nullptr,
            cudaEvent_t after_up = nullptr) {
  const int n_blk = (T + kBlockTokens - 1) / kBlockTokens;
  PlanArgs pa{};
  pa.T = T;
  pa.d = d;
  pa.f_local = f_local;
  pa.rc_local = has_comp ? rc_local : 0;
  pa.n_blk = n_blk;
  pa.sparse_begin = sparse_begin;
  pa.sparse_count = sparse_count;
  pa.k_shared = k_shared;
  pa.counts = counts;
  pa.idx_shared = idx_shared;
  pa.has_comp = has_comp;
  pa.up_group = g_up_group.load(std::memory_order_relaxed);
  pa.down_group = g_down_group.load(std::memory_order_relaxed);
  pa.bn_down = bn_for(d);
  pa.hcols_alloc = w.hcols;
  pa.serpentine = g_serpentine.load(std::memory_order_relaxed);
  pa.pair_up = up_proj_paired() ? 1 : 0;
  pa.pair_down = down_proj_paired() ? 1 : 0;
  pa.blk_done = (g_blockdep.load(std::memory_order_relaxed) && !up_only) ? w.blk_done : nullptr;
  {
    StageTimer tm(kPlan, s);
    FFWD_CUDA(launch_plan(pa, w.meta, w.up, w.up_cap, w.down, w.down_cap, w.pc, s), "plan");
  }
  GemmArgs ga{};
  ga.x = x;
  ga.wgu_t = wgu_t;
  ga.wgu_rows = 2 * f_local + rup(rc_local, 256);
  ga.wd = wd;
  ga.wd_rows = f_local + rup(rc_local, 64);
  ga.h = w.h;
  ga.hcols = w.hcols;
  ga.y = y;
  ga.residual = residual;
  ga.x_next = x_next;
  ga.T = T;
  ga.d = d;
  ga.f_local = f_local;
  ga.n_blk = n_blk;
  ga.idx = idx;
  ga.ld_idx = ld_idx;
  ga.meta = w.meta;
  ga.up_tiles = w.up;
  ga.up_cap = w.up_cap;
  ga.down_tiles = w.down;
  ga.down_cap = w.down_cap;
  ga.counts = w.pc;
  ga.num_sms = num_sms();
  ga.bn_down = bn_for(d);
  ga.blk_done = pa.blk_done;
  ga.y_done = y_done;
  {
    StageTimer tm(kUp, s);
    FFWD_CUDA(launch_up_proj(ga, s), "up_proj");
  }
  if (up_only) return FFWD_OK;  // H only (oracle scoring)
  if (after_up) FFWD_CUDA(cudaEventRecord(after_up, s), "event record");
  {
    StageTimer tm(kDown, s);
    FFWD_CUDA(launch_down_proj(ga, s), "down_proj");
  }
  return FFWD_OK;
}

int check_gemm_shapes(int d, int f_local) {
  if (d % 64 != 0)
    return fail(FFWD_ERR_UNSUPPORTED, "d_model=%d: the sm_100a path needs d_model %% 64 == 0", d);
  if (f_local < 1) return fail(FFWD_ERR_VALIDATION, "f_local must be >= 1");
  return FFWD_OK;
}

}  // namespace

namespace ffwd {
bool pdl_enabled() { return g_pdl.load(std::memory_order_relaxed) != 0; }
unsigned long long spin_timeout_ns() {
  return static_cast<unsigned long long>(g_spin_timeout_ms.load(std::memory_order_relaxed)) *
         1000000ull;
}
}  // namespace ffwd

extern "C" {

int ffwd_abi_version(void) { return FFWD_ABI_VERSION; }

const char* ffwd_last_error(void) { return g_err.c_str(); }

int ffwd_device_check(int device) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (p.major != 10 || p.minor != 0)
    return fail(FFWD_ERR_UNSUPPORTED, "device %d is sm_%d%d; kernels are built for sm_100a",
                device, p.major, p.minor);
  return FFWD_OK;
}

int ffwd_set_pdl(int on) {
  g_pdl = on != 0;
  return FFWD_OK;
}

int ffwd_set_spin_timeout_ms(int ms) {
  if (ms < 1) return fail(FFWD_ERR_VALIDATION, "spin timeout must be >= 1 ms, got %d", ms);
  g_spin_timeout_ms.store(ms);
  return FFWD_OK;
}

int ffwd_set_serpentine(int on) {
  g_serpentine = on != 0;
  return FFWD_OK;
}

int ffwd_set_raster(int up_group, int down_group) {
  if (up_group < 1 || down_group < 1)
    return fail(FFWD_ERR_VALIDATION, "raster groups must be >= 1");
  g_up_group.store(up_group);
  g_down_group.store(down_group);
  return FFWD_OK;
}

size_t ffwd_predictor_workspace_bytes(int blk_count, int d, int r, int f) {
  Carve c(nullptr);
  carve_pred(c, blk_count, d, r, f, false);
  return c.off;
}

int ffwd_predictor_forward(const void* x, int x_is_f32, int T, int d, int blk_begin,
                           int blk_count, const float* query, const float* w1, const float* w2,
                           int r, int f, float* scores, void* workspace, size_t workspace_bytes,
                           void* stream) {
  g_err.clear();
  if (T < 1 || d < 1 || r < 1 || f < 1)
    return fail(FFWD_ERR_VALIDATION, "predictor dims T=%d d=%d r=%d f=%d", T, d, r, f);
  if (!x || !query || !w1 || !w2 || !scores || (blk_count > 0 && !workspace))
    return fail(FFWD_ERR_VALIDATION, "predictor_forward: null pointer");
  const int n_blk = (T + kBlockTokens - 1) / kBlockTokens;
  if (blk_begin < 0 || blk_count < 0 || blk_begin + blk_count > n_blk)
    return fail(FFWD_ERR_VALIDATION, "block range [%d, %d) outside [0, %d)", blk_begin,
                blk_begin + blk_count, n_blk);
  if (workspace_bytes < ffwd_predictor_workspace_bytes(blk_count, d, r, f))
    return fail(FFWD_ERR_VALIDATION, "workspace too small");
  Carve c(workspace);
  Pred p = carve_pred(c, blk_count, d, r, f, false);
  return run_predictor(x, x_is_f32 != 0, T, d, blk_begin, blk_count, query, w1, w2, r, f, p,
                       scores, static_cast<cudaStream_t>(stream));
}

int ffwd_predictor_forward_block(const void* x, int x_is_f32, int n, int d, const float* query,
                                 const float* w1, const float* w2, int r, int f, float* scores,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (n < 1 || d < 1 || r < 1 || f < 1)
    return fail(FFWD_ERR_VALIDATION, "predictor dims n=%d d=%d r=%d f=%d", n, d, r, f);
  if (n > 25600)
    return fail(FFWD_ERR_UNSUPPORTED, "predictor_forward_block: n=%d > 25600 rows", n);
  if (!x || !query || !w1 || !w2 || !scores || !workspace)
    return fail(FFWD_ERR_VALIDATION, "predictor_forward_block: null pointer");
  if (workspace_bytes < ffwd_predictor_workspace_bytes(1, d, r, f))
    return fail(FFWD_ERR_VALIDATION, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carve c(workspace);
  Pred p = carve_pred(c, 1, d, r, f, false);
  const float sqrt_d = static_cast<float>(std::sqrt(static_cast<double>(d)));  // predictor.py:76
  FFWD_CUDA(launch_pool_generic(x, x_is_f32 != 0, n, d, n, 0, 1, query, sqrt_d, p.pooled, s),
            "pool");
  FFWD_CUDA(launch_gemm_f64acc(p.pooled, w1, p.hidden, 1, d, r, true, p.partial, s), "w1");
  FFWD_CUDA(launch_gemm_f64acc(p.hidden, w2, scores, 1, r, f, false, nullptr, s), "w2");
  return FFWD_OK;
}

int ffwd_predictor_logits(const void* x, int x_is_f32, int T, int d, const float* query,
                          float* logits, void* stream) {
  g_err.clear();
  if (!x || !query || !logits) return fail(FFWD_ERR_VALIDATION, "predictor_logits: null pointer");
  if (T < 1 || d < 4 || d % 4 != 0)
    return fail(FFWD_ERR_VALIDATION, "predictor_logits dims T=%d d=%d (d %% 4 == 0)", T, d);
  if (d > 16384) return fail(FFWD_ERR_UNSUPPORTED, "predictor_logits: d_model <= 16384");
  const float sqrt_d = static_cast<float>(std::sqrt(static_cast<double>(d)));  // predictor.py:76
  FFWD_CUDA(launch_logits_only(x, x_is_f32 != 0, d, 0, T, query, sqrt_d, logits,
                               static_cast<cudaStream_t>(stream)),
            "predictor_logits");
  return FFWD_OK;
}

int ffwd_topk(const float* scores, int n_rows, int f, int k, int tp_rank, int tp_size,
              int32_t* idx_global, int ld_global, int32_t* idx_local, int ld_local,
              int32_t* counts, void* stream) {
  g_err.clear();
  if (n_rows < 0 || f < 1) return fail(FFWD_ERR_VALIDATION, "bad top-k shape");
  if (k < 1 || k > f) return fail(FFWD_ERR_VALIDATION, "k=%d out of range [1, %d]", k, f);
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size)
    return fail(FFWD_ERR_VALIDATION, "bad tensor-parallel rank %d of %d", tp_rank, tp_size);
  if (idx_global && ld_global < k) return fail(FFWD_ERR_VALIDATION, "ld_global < k");
  if (n_rows > 0 && (!scores || (!idx_global && !idx_local)))
    return fail(FFWD_ERR_VALIDATION, "topk: null scores or no index output");
  if (idx_local && ld_local < std::min(k, (f + tp_size - 1) / tp_size))
    return fail(FFWD_ERR_VALIDATION, "ld_local too small");
  FFWD_CUDA(launch_topk(scores, n_rows, f, k, tp_rank, tp_size, idx_global, ld_global, idx_local,
                        ld_local, counts, static_cast<cudaStream_t>(stream)),
            "topk");
  return FFWD_OK;
}

int ffwd_predict_topk(const void* x, int x_is_f32, int T, int d, int blk_begin, int blk_count,
                      const float* query, const float* w1, const float* w2, int r, int f, int k,
                      int tp_rank, int tp_size, int32_t* idx_global, int ld_global,
                      int32_t* idx_local, int ld_local, int32_t* counts, void* workspace,
                      size_t workspace_bytes, void* stream) {
  const size_t pred_bytes = ffwd_predictor_workspace_bytes(blk_count, d, r, f);
  const size_t need = pred_bytes + al(static_cast<size_t>(blk_count) * f * sizeof(float));
  if (workspace_bytes < need) return fail(FFWD_ERR_VALIDATION, "workspace too small");
  float* scores = reinterpret_cast<float*>(static_cast<char*>(workspace) + pred_bytes);
  int rc = ffwd_predictor_forward(x, x_is_f32, T, d, blk_begin, blk_count, query, w1, w2, r, f,
                                  scores, workspace, workspace_bytes, stream);
  if (rc != FFWD_OK) return rc;
  return ffwd_topk(scores, blk_count, f, k, tp_rank, tp_size, idx_global, ld_global, idx_local,
                   ld_local, counts, stream);
}

size_t ffwd_sparse_ffn_workspace_bytes(int T, int d, int f_local, int rc_local, int k) {
  Carve c(nullptr);
  carve_ffn(c, T, d, f_local, rc_local, k, 0, 4);
  return c.off;
}

int ffwd_sparse_ffn(const void* x_bf16, int T, int d, const void* wgu_t, const void* wd,
                    int f_local, int rc_local, const int32_t* idx, int idx_per_block, int ld_idx,
                    const int32_t* counts, int k, int has_comp, float* y, void* workspace,
                    size_t workspace_bytes, void* stream) {
  g_err.clear();
  int rc = check_common(T, d, f_local, k);
  if (rc) return rc;
  if ((rc = check_gemm_shapes(d, f_local))) return rc;
  if (has_comp && rc_local < 1) return fail(FFWD_ERR_VALIDATION, "compensator width must be >= 1");
  if (!x_bf16 || !wgu_t || !wd || !y || !workspace)
    return fail(FFWD_ERR_VALIDATION, "sparse_ffn: null pointer");
  if (idx && ld_idx < k) return fail(FFWD_ERR_VALIDATION, "ld_idx < k");
  if (workspace_bytes < ffwd_sparse_ffn_workspace_bytes(T, d, f_local, rc_local, k))
    return fail(FFWD_ERR_VALIDATION, "workspace too small");
  Carve c(workspace);
  Ffn w = carve_ffn(c, T, d, f_local, rc_local, k, 0, 4);
  const int n_blk = (T + kBlockTokens - 1) / kBlockTokens;
  if (idx == nullptr)  // dense_ffn: identity over every neuron
    return run_ffn(x_bf16, T, d, wgu_t, wd, f_local, rc_local, w, nullptr, 0, 0, 0, nullptr,
                   f_local, 0, 0, y, nullptr, nullptr, static_cast<cudaStream_t>(stream));
  return run_ffn(x_bf16, T, d, wgu_t, wd, f_local, rc_local, w, idx, ld_idx, 0, n_blk, counts, k,
                 idx_per_block ? 0 : 1, has_comp, y, nullptr, nullptr,
                 static_cast<cudaStream_t>(stream));
}

static void layer_split(int T, int k, int f_global, int dense_first_last, int* begin,
                        int* count) {
  const int n_blk = (T + kBlockTokens - 1) / kBlockTokens;
  if (k >= f_global) {  // engine.py:268 full-K shortcut: every block dense
    *begin = 0;
    *count = 0;
  } else if (dense_first_last) {  // engine.py:258-262
    // 1: the whole prompt (first and last block dense); 2 / 3: a sequence shard holding
    // only the prompt's first / only its last block
    const int first = dense_first_last != 3 ? 1 : 0, last = dense_first_last != 2 ? 1 : 0;
    *begin = first;
    *count = n_blk > first + last ? n_blk - first - last : 0;
  } else {
    *begin = 0;
    *count = n_blk;
  }
}

static int local_kmax(int k, int f_local) { return k < f_local ? k : f_local; }

size_t ffwd_layer_workspace_bytes(int T, int d, int f_global, int f_local, int rc_local, int r,
                                  int k, int dense_first_last, int tp_size) {
  int b0, nb;
  layer_split(T, k, f_global, dense_first_last, &b0, &nb);
  (void)tp_size;
  const int kmax = local_kmax(k, f_local);
  Carve c(nullptr);
  carve_pred(c, nb, d, r, f_global, true);
  carve_ffn(c, T, d, f_local, rc_local, kmax, nb, rup(kmax, 4));
  return c.off;
}

int ffwd_ffn_layer2(const void* x_bf16, int T, int d, const void* wgu_t, const void* wd,
                    int f_local, int rc_local, const float* query, const float* w1,
                    const float* w2, int r, int f_global, int k, int dense_first_last,
                    int has_comp, int tp_rank, int tp_size, float* y, const float* residual,
                    void* x_next_bf16, int32_t* idx_global, int ld_idx_global,
                    const float* x_pred_f32, const float* logits_in, void* workspace,
                    size_t workspace_bytes, void* stream) {
  g_err.clear();
  int rc = check_common(T, d, f_global, k);
  if (rc) return rc;
  if ((rc = check_gemm_shapes(d, f_local))) return rc;
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size)
    return fail(FFWD_ERR_VALIDATION, "bad tensor-parallel rank %d of %d", tp_rank, tp_size);
  if (dense_first_last < 0 || dense_first_last > 3)
    return fail(FFWD_ERR_VALIDATION, "dense_first_last must be 0..3, got %d", dense_first_last);
  if (f_local != (f_global - tp_rank + tp_size - 1) / tp_size)
    return fail(FFWD_ERR_VALIDATION, "f_local=%d is not rank %d's strided share of d_ffn=%d",
                f_local, tp_rank, f_global);
  if (has_comp && rc_local < 1) return fail(FFWD_ERR_VALIDATION, "compensator width must be >= 1");
  if (residual && tp_size != 1)
    return fail(FFWD_ERR_VALIDATION, "fused residual needs tp_size == 1 (reduce the partials first)");
  if (!x_bf16 || !wgu_t || !wd || !workspace || (!y && !x_next_bf16))
    return fail(FFWD_ERR_VALIDATION, "ffn_layer: null x, weight, output or workspace pointer");
  if (!y && residual)
    return fail(FFWD_ERR_VALIDATION, "ffn_layer: the residual add needs the f32 output y");
  if (workspace_bytes <
      ffwd_layer_workspace_bytes(T, d, f_global, f_local, rc_local, r, k, dense_first_last, tp_size))
    return fail(FFWD_ERR_VALIDATION, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int b0, nb;
  layer_split(T, k, f_global, dense_first_last, &b0, &nb);
  if (nb > 0 && (!query || !w1 || !w2))
    return fail(FFWD_ERR_VALIDATION, "ffn_layer: predicted blocks need the predictor weights");
  const int kmax = local_kmax(k, f_local);
  Carve c(workspace);
  Pred p = carve_pred(c, nb, d, r, f_global, true);
  Ffn w = carve_ffn(c, T, d, f_local, rc_local, kmax, nb, rup(kmax, 4));
  if (nb > 0) {
    if (d % 8 != 0) return fail(FFWD_ERR_UNSUPPORTED, "predictor needs d_model %% 8 == 0");
    if (idx_global && ld_idx_global < k) return fail(FFWD_ERR_VALIDATION, "ld_idx_global < k");
    rc = x_pred_f32 ? run_predictor(x_pred_f32, true, T, d, b0, nb, query, w1, w2, r, f_global,
                                    p, p.scores, s, logits_in)
                    : run_predictor(x_bf16, false, T, d, b0, nb, query, w1, w2, r, f_global, p,
                                    p.scores, s, logits_in);
    if (rc) return rc;
    {
      StageTimer tm(kTopk, s);
      FFWD_CUDA(launch_topk(p.scores, nb, f_global, k, tp_rank, tp_size, idx_global,
                            ld_idx_global, w.idx_local, w.ld_local, w.counts, s),
                "topk");
    }
  }
  return run_ffn(x_bf16, T, d, wgu_t, wd, f_local, rc_local, w, w.idx_local, w.ld_local, b0, nb,
                 tp_size > 1 ? w.counts : nullptr, k, 0, has_comp, y, residual, x_next_bf16, s);
}

size_t ffwd_predict_mask_workspace_bytes(int blk_count, int d, int r, int f) {
  Carve c(nullptr);
  carve_pred(c, blk_count, d, r, f, true);
  return c.off;
}

int ffwd_predict_mask(const void* x, int x_is_f32, int T, int d, int blk_begin, int blk_count,
                      const float* query, const float* w1, const float* w2, int r, int f, int k,
                      const float* logits_in, uint32_t* mask, int ld_mask, void* workspace,
                      size_t workspace_bytes, void* stream) {
  g_err.clear();
  int rc = check_common(T, d, f, k);
  if (rc) return rc;
  if (blk_count < 1 || blk_begin < 0 || (blk_begin + blk_count - 1) * kBlockTokens >= T)
    return fail(FFWD_ERR_VALIDATION, "blocks [%d, %d) outside the %d tokens", blk_begin,
                blk_begin + blk_count, T);
  if (d % 8 != 0) return fail(FFWD_ERR_UNSUPPORTED, "predictor needs d_model %% 8 == 0");
  if (ld_mask < (f + 31) / 32) return fail(FFWD_ERR_VALIDATION, "ld_mask < ceil(f / 32)");
  if (!x || !query || !w1 || !w2 || !mask || !workspace)
    return fail(FFWD_ERR_VALIDATION, "predict_mask: null pointer");
  if (workspace_bytes < ffwd_predict_mask_workspace_bytes(blk_count, d, r, f))
    return fail(FFWD_ERR_VALIDATION, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carve c(workspace);
  Pred p = carve_pred(c, blk_count, d, r, f, true);
  rc = run_predictor(x, x_is_f32 != 0, T, d, blk_begin, blk_count, query, w1, w2, r, f, p,
                     p.scores, s, logits_in);
  if (rc) return rc;
  StageTimer tm(kTopk, s);
  FFWD_CUDA(launch_topk(p.scores, blk_count, f, k, 0, 1, nullptr, 0, nullptr, 0, nullptr, s, mask,
                        ld_mask),
            "topk");
  return FFWD_OK;
}

int ffwd_ffn_layer_masked(const void* x_bf16, int T, int d, const void* wgu_t, const void* wd,
                          int f_local, int rc_local, int f_global, int k, int dense_first_last,
                          int has_comp, int tp_rank, int tp_size, const uint32_t* mask,
                          int ld_mask, float* y, const float* residual, void* x_next_bf16,
                          void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  int rc = check_common(T, d, f_global, k);
  if (rc) return rc;
  if ((rc = check_gemm_shapes(d, f_local))) return rc;
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size)
    return fail(FFWD_ERR_VALIDATION, "bad tensor-parallel rank %d of %d", tp_rank, tp_size);
  if (dense_first_last < 0 || dense_first_last > 3)
    return fail(FFWD_ERR_VALIDATION, "dense_first_last must be 0..3, got %d", dense_first_last);
  if (f_local != (f_global - tp_rank + tp_size - 1) / tp_size)
    return fail(FFWD_ERR_VALIDATION, "f_local=%d is not rank %d's strided share of d_ffn=%d",
                f_local, tp_rank, f_global);
  if (has_comp && rc_local < 1) return fail(FFWD_ERR_VALIDATION, "compensator width must be >= 1");
  if (residual && tp_size != 1)
    return fail(FFWD_ERR_VALIDATION, "fused residual needs tp_size == 1 (reduce the partials first)");
  if (!x_bf16 || !wgu_t || !wd || !workspace || (!y && !x_next_bf16))
    return fail(FFWD_ERR_VALIDATION, "ffn_layer: null x, weight, output or workspace pointer");
  if (!y && residual)
    return fail(FFWD_ERR_VALIDATION, "ffn_layer: the residual add needs the f32 output y");
  int b0, nb;
  layer_split(T, k, f_global, dense_first_last, &b0, &nb);
  if (nb > 0 && (!mask || ld_mask < (f_global + 31) / 32))
    return fail(FFWD_ERR_VALIDATION, "ffn_layer_masked: predicted blocks need mask rows of "
                "ceil(d_ffn / 32) words");
  const int kmax = local_kmax(k, f_local);
  Carve c0(nullptr);
  carve_ffn(c0, T, d, f_local, rc_local, kmax, nb, rup(kmax, 4));
  if (workspace_bytes < c0.off) return fail(FFWD_ERR_VALIDATION, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carve c(workspace);
  Ffn w = carve_ffn(c, T, d, f_local, rc_local, kmax, nb, rup(kmax, 4));
  if (nb > 0) {
    StageTimer tm(kTopk, s);
    FFWD_CUDA(launch_mask_to_local(mask + static_cast<size_t>(b0) * ld_mask, ld_mask, nb,
                                   f_global, tp_rank, tp_size, w.idx_local, w.ld_local, w.counts,
                                   s),
              "mask_to_local");
  }
  return run_ffn(x_bf16, T, d, wgu_t, wd, f_local, rc_local, w, w.idx_local, w.ld_local, b0, nb,
                 w.counts, k, 0, has_comp, y, residual, x_next_bf16, s);
}

int ffwd_ffn_layer(const void* x_bf16, int T, int d, const void* wgu_t, const void* wd,
                   int f_local, int rc_local, const float* query, const float* w1,
                   const float* w2, int r, int f_global, int k, int dense_first_last,
                   int has_comp, int tp_rank, int tp_size, float* y, const float* residual,
                   void* x_next_bf16, int32_t* idx_global, int ld_idx_global, void* workspace,
                   size_t workspace_bytes, void* stream) {
  return ffwd_ffn_layer2(x_bf16, T, d, wgu_t, wd, f_local, rc_local, query, w1, w2, r, f_global,
                         k, dense_first_last, has_comp, tp_rank, tp_size, y, residual,
                         x_next_bf16, idx_global, ld_idx_global, nullptr, nullptr, workspace,
                         workspace_bytes, stream);
}

size_t ffwd_hidden_scores_workspace_bytes(int T, int d, int f) {
  Carve c(nullptr);
  carve_ffn(c, T, d, f, 0, f, 0, 4);
  return c.off;
}

int ffwd_hidden_scores(const void* x_bf16, int T, int d, const void* wgu_t, int f,
                       int rc_local, float* scores, void* workspace, size_t workspace_bytes,
                       void* stream) {
  g_err.clear();
  int rc = check_common(T, d, f, f);
  if (rc) return rc;
  if ((rc = check_gemm_shapes(d, f))) return rc;
  if (!x_bf16 || !wgu_t || !scores || !workspace)
    return fail(FFWD_ERR_VALIDATION, "hidden_scores: null pointer");
  if (workspace_bytes < ffwd_hidden_scores_workspace_bytes(T, d, f))
    return fail(FFWD_ERR_VALIDATION, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carve c(workspace);
  Ffn w = carve_ffn(c, T, d, f, 0, f, 0, 4);
  // dense gate/up over every block (identity index, no compensator): H = silu(g) * u
  rc = run_ffn(x_bf16, T, d, wgu_t, nullptr, f, rc_local, w, nullptr, 0, 0, 0, nullptr, f, 0, 0,
               nullptr, nullptr, nullptr, s, /*up_only=*/true);
  if (rc) return rc;
  FFWD_CUDA(launch_hidden_scores(w.h, false, w.hcols, T, f, kBlockTokens, scores, s),
            "hidden_scores");
  return FFWD_OK;
}

int ffwd_column_norms(const void* h, int is_f32, int n_rows, int ld, int f, float* scores,
                      void* stream) {
  g_err.clear();
  if (n_rows < 1 || f < 1 || ld < f)
    return fail(FFWD_ERR_VALIDATION, "column_norms dims n=%d f=%d ld=%d", n_rows, f, ld);
  if (!h || !scores) return fail(FFWD_ERR_VALIDATION, "column_norms: null pointer");
  // one block of all n_rows rows (sparse.py:94-97 scores whatever block it is given)
  FFWD_CUDA(launch_hidden_scores(h, is_f32 != 0, ld, n_rows, f, n_rows, scores,
                                 static_cast<cudaStream_t>(stream)),
            "column_norms");
  return FFWD_OK;
}

size_t ffwd_ffn_layer_mode_workspace_bytes(int T, int d, int f, int rc_local, int k, int mode,
                                           int dense_first_last) {
  const int n_blk = (T + kBlockTokens - 1) / kBlockTokens;
  int b0 = 0, nb = 0;
  layer_split(T, k, f, dense_first_last || mode == 2, &b0, &nb);
  if (mode == 2 && !dense_first_last && k < f) nb = n_blk - 1;  // static: only block 0 dense
  const int n_score = mode == 2 ? 1 : nb;
  const int t_score = std::max(1, std::min(T - (mode == 2 ? 0 : b0) * kBlockTokens,
                                           n_score * kBlockTokens));
  Carve c(nullptr);
  c.take<float>(static_cast<size_t>(std::max(1, n_score)) * f);           // scores
  c.take<int32_t>(static_cast<size_t>(std::max(1, n_score)) * rup(k, 4));  // indices
  const size_t a = c.off + ffwd_hidden_scores_workspace_bytes(t_score, d, f);
  Carve c2(nullptr);
  carve_ffn(c2, T, d, f, rc_local, k, 0, 4);
  return std::max(a, c.off + c2.off);
}

int ffwd_ffn_layer_mode(const void* x_bf16, int T, int d, const void* wgu_t, const void* wd,
                        int f, int rc_local, int k, int mode, int dense_first_last, int has_comp,
                        float* y, const float* residual, void* x_next_bf16, int32_t* idx_out,
                        int ld_idx_out, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  int rc = check_common(T, d, f, k);
  if (rc) return rc;
  if ((rc = check_gemm_shapes(d, f))) return rc;
  if (mode != 1 && mode != 2)
    return fail(FFWD_ERR_VALIDATION, "mode %d: expected 1 (oracle) or 2 (static)", mode);
  if (dense_first_last != 0 && dense_first_last != 1)
    return fail(FFWD_ERR_VALIDATION, "ablation modes take dense_first_last 0 or 1");
  if (has_comp && rc_local < 1) return fail(FFWD_ERR_VALIDATION, "compensator width must be >= 1");
  if (!x_bf16 || !wgu_t || !wd || !y || !workspace)
    return fail(FFWD_ERR_VALIDATION, "ffn_layer_mode: null pointer");
  if (workspace_bytes <
      ffwd_ffn_layer_mode_workspace_bytes(T, d, f, rc_local, k, mode, dense_first_last))
    return fail(FFWD_ERR_VALIDATION, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n_blk = (T + kBlockTokens - 1) / kBlockTokens;
  int b0 = 0, nb = 0;
  // engine.py:256-262: dense if dense_first_last and j in {0, last}, or static and j == 0
  layer_split(T, k, f, dense_first_last || mode == 2, &b0, &nb);
  if (mode == 2 && !dense_first_last && k < f) nb = n_blk - 1;
  if (idx_out && ld_idx_out < k) return fail(FFWD_ERR_VALIDATION, "ld_idx_out < k");
  if (k >= f)  // full-K shortcut (engine.py:268): every block dense, no masks
    return run_ffn(x_bf16, T, d, wgu_t, wd, f, rc_local, carve_ffn_at(workspace, T, d, f,
                   rc_local, k), nullptr, 0, 0, 0, nullptr, f, 0, 0, y, residual, x_next_bf16, s);
  // static scores block 0 even when no later block is sparse (the reference still
  // records its mask, engine.py:273-277)
  const int n_score = mode == 2 ? 1 : nb;
  const int s_blk0 = mode == 2 ? 0 : b0;  // first scored block
  Carve c(workspace);
  float* scores = c.take<float>(static_cast<size_t>(std::max(1, n_score)) * f);
  const int ld = rup(k, 4);
  int32_t* idx = c.take<int32_t>(static_cast<size_t>(std::max(1, n_score)) * ld);
  const size_t off = c.off;
  if (n_score > 0) {
    const int t_score = std::min(T - s_blk0 * kBlockTokens, n_score * kBlockTokens);
    // 1. dense gate/up of the scored blocks -> column norms (sparse.py:94-115 oracle_experts
    //    / mask_from_hidden); counted like the reference (costmodel oracle: 4 n d f)
    rc = ffwd_hidden_scores(static_cast<const __nv_bfloat16*>(x_bf16) +
                                static_cast<size_t>(s_blk0) * kBlockTokens * d,
                            t_score, d, wgu_t, f, rc_local, scores,
                            static_cast<char*>(workspace) + off, workspace_bytes - off, stream);
    if (rc) return rc;
    // 2. top-k of the scores (build_mask)
    FFWD_CUDA(launch_topk(scores, n_score, f, k, 0, 1, nullptr, 0, idx, ld, nullptr, s), "topk");
    if (idx_out)
      FFWD_CUDA(cudaMemcpy2DAsync(idx_out, static_cast<size_t>(ld_idx_out) * 4, idx,
                                  static_cast<size_t>(ld) * 4, static_cast<size_t>(k) * 4,
                                  n_score, cudaMemcpyDeviceToDevice, s),
                "idx copy");
  }
  if (nb == 0)  // no sparse block: the dense FFN over every block
    return run_ffn(x_bf16, T, d, wgu_t, wd, f, rc_local,
                   carve_ffn_at(static_cast<char*>(workspace) + off, T, d, f, rc_local, k),
                   nullptr, 0, 0, 0, nullptr, f, 0, 0, y, residual, x_next_bf16, s);
  // 3. sparse FFN (+ compensator) with those masks; static: one mask for every block
  Carve c2(static_cast<char*>(workspace) + off);
  Ffn w = carve_ffn(c2, T, d, f, rc_local, k, 0, 4);
  return run_ffn(x_bf16, T, d, wgu_t, wd, f, rc_local, w, idx, ld, b0, nb, nullptr, k,
                 mode == 2 ? 1 : 0, has_comp, y, residual, x_next_bf16, s);
}

int ffwd_ipc_get_handle(void* dev_ptr, void* handle_out, size_t* offset_out) {
  g_err.clear();
  // the handle names the whole allocation; the opener adds this pointer's offset
  using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      return fail(FFWD_ERR_CUDA, "cuMemGetAddressRange unavailable");
    range = reinterpret_cast<RangeFn>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(FFWD_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  FFWD_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = static_cast<size_t>(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return FFWD_OK;
}

int ffwd_ipc_open(const void* handle, void** dev_ptr) {
  g_err.clear();
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  FFWD_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess),
            "cudaIpcOpenMemHandle");
  return FFWD_OK;
}

int ffwd_ipc_close(void* dev_ptr) {
  g_err.clear();
  FFWD_CUDA(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
  return FFWD_OK;
}

int ffwd_allreduce_residual(const float* const* partials, float* const* outs,
                            void* const* xnexts, unsigned* const* flags, int n_ranks, int rank,
                            const float* residual, int T, int d, unsigned epoch, int max_ctas,
                            void* stream) {
  g_err.clear();
  if (n_ranks < 1 || n_ranks > 8 || rank < 0 || rank >= n_ranks)
    return fail(FFWD_ERR_VALIDATION, "bad rank %d of %d (1..8 ranks)", rank, n_ranks);
  if (T < 1 || d < 4 || d % 4 != 0)
    return fail(FFWD_ERR_VALIDATION, "allreduce dims T=%d d=%d (d %% 4 == 0)", T, d);
  if (!partials || !outs || !flags || !residual)
    return fail(FFWD_ERR_VALIDATION, "allreduce needs partial, out, flag and residual pointers");
  for (int p = 0; p < n_ranks; ++p)
    if (!partials[p] || !outs[p] || !flags[p] || (xnexts && !xnexts[p]))
      return fail(FFWD_ERR_VALIDATION, "null peer pointer for rank %d", p);
  const int ctas = max_ctas > 0 ? max_ctas : num_sms();
  FFWD_CUDA(launch_allreduce_residual(partials, outs, xnexts, flags, n_ranks, rank, residual, T,
                                      d, epoch, ctas, static_cast<cudaStream_t>(stream)),
            "allreduce_residual");
  return FFWD_OK;
}

int ffwd_ffn_layer_tp_overlap(const void* x_bf16, int T, int d, const void* wgu_t,
                              const void* wd, int f_local, int rc_local, const float* query,
                              const float* w1, const float* w2, int r, int f_global, int k,
                              int dense_first_last, int has_comp, int tp_rank, int tp_size,
                              int32_t* idx_global, int ld_idx_global, const float* x_pred_f32,
                              const float* logits_in, const float* const* partials,
                              float* const* outs, void* const* xnexts, unsigned* const* flags,
                              unsigned* const* y_done, const float* residual, unsigned epoch,
                              unsigned y_epoch, int comm_ctas, void* workspace,
                              size_t workspace_bytes, void* stream, void* comm_stream) {
  g_err.clear();
  int rc = check_common(T, d, f_global, k);
  if (rc) return rc;
  if ((rc = check_gemm_shapes(d, f_local))) return rc;
  if (tp_size < 1 || tp_size > 8 || tp_rank < 0 || tp_rank >= tp_size)
    return fail(FFWD_ERR_VALIDATION, "bad tensor-parallel rank %d of %d (1..8 ranks)", tp_rank,
                tp_size);
  if (dense_first_last < 0 || dense_first_last > 3)
    return fail(FFWD_ERR_VALIDATION, "dense_first_last must be 0..3, got %d", dense_first_last);
  if (f_local != (f_global - tp_rank + tp_size - 1) / tp_size)
    return fail(FFWD_ERR_VALIDATION, "f_local=%d is not rank %d's strided share of d_ffn=%d",
                f_local, tp_rank, f_global);
  if (has_comp && rc_local < 1) return fail(FFWD_ERR_VALIDATION, "compensator width must be >= 1");
  if (!partials || !outs || !flags || !y_done || !residual)
    return fail(FFWD_ERR_VALIDATION,
                "overlapped completion needs partial, out, flag, y_done and residual pointers");
  if (!x_bf16 || !wgu_t || !wd || !workspace)
    return fail(FFWD_ERR_VALIDATION, "ffn_layer_tp_overlap: null x, weight or workspace pointer");
  for (int p = 0; p < tp_size; ++p)
    if (!partials[p] || !outs[p] || !flags[p] || !y_done[p] || (xnexts && !xnexts[p]))
      return fail(FFWD_ERR_VALIDATION, "null peer pointer for rank %d", p);
  if (xnexts && xnexts[tp_rank] == x_bf16)
    return fail(FFWD_ERR_VALIDATION, "x_next must not alias the layer input (peers write it "
                                     "while this rank may still read it)");
  if (workspace_bytes <
      ffwd_layer_workspace_bytes(T, d, f_global, f_local, rc_local, r, k, dense_first_last, tp_size))
    return fail(FFWD_ERR_VALIDATION, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t cs = static_cast<cudaStream_t>(comm_stream);
  if (cs == s) return fail(FFWD_ERR_VALIDATION, "the completion needs its own stream");
  // events belong to a device: one pair per (thread, device)
  static thread_local cudaEvent_t evs[64][2] = {};
  int dev = 0;
  FFWD_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  cudaEvent_t& ev_up = evs[dev & 63][0];
  cudaEvent_t& ev_done = evs[dev & 63][1];
  if (!ev_up) {
    FFWD_CUDA(cudaEventCreateWithFlags(&ev_up, cudaEventDisableTiming), "event create");
    FFWD_CUDA(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming), "event create");
  }
  int b0, nb;
  layer_split(T, k, f_global, dense_first_last, &b0, &nb);
  const int kmax = local_kmax(k, f_local);
  Carve c(workspace);
  Pred p = carve_pred(c, nb, d, r, f_global, true);
  Ffn w = carve_ffn(c, T, d, f_local, rc_local, kmax, nb, rup(kmax, 4));
  if (nb > 0) {
    if (d % 8 != 0) return fail(FFWD_ERR_UNSUPPORTED, "predictor needs d_model %% 8 == 0");
    if (idx_global && ld_idx_global < k) return fail(FFWD_ERR_VALIDATION, "ld_idx_global < k");
    rc = x_pred_f32 ? run_predictor(x_pred_f32, true, T, d, b0, nb, query, w1, w2, r, f_global,
                                    p, p.scores, s, logits_in)
                    : run_predictor(x_bf16, false, T, d, b0, nb, query, w1, w2, r, f_global, p,
                                    p.scores, s, logits_in);
    if (rc) return rc;
    StageTimer tm(kTopk, s);
    FFWD_CUDA(launch_topk(p.scores, nb, f_global, k, tp_rank, tp_size, idx_global, ld_idx_global,
                          w.idx_local, w.ld_local, w.counts, s),
              "topk");
  }
  // K3 publishes per-block tile counts; the completion starts once K2 retired (its CTAs
  // then sit beside K3's, one K3 CTA per SM leaving the room) and drains blocks as they
  // finish on every rank
  rc = run_ffn(x_bf16, T, d, wgu_t, wd, f_local, rc_local, w, w.idx_local, w.ld_local, b0, nb,
               tp_size > 1 ? w.counts : nullptr, k, 0, has_comp,
               const_cast<float*>(partials[tp_rank]), nullptr, nullptr, s, false,
               y_done[tp_rank], ev_up);
  if (rc) return rc;
  FFWD_CUDA(cudaStreamWaitEvent(cs, ev_up, 0), "stream wait");
  const unsigned target = y_epoch * static_cast<unsigned>(d / bn_for(d));
  FFWD_CUDA(launch_allreduce_overlap(partials, outs, xnexts, flags, y_done, tp_size, tp_rank,
                                     residual, T, d, epoch, target, b0, nb,
                                     comm_ctas > 0 ? comm_ctas : 32, cs),
            "allreduce_overlap");
  FFWD_CUDA(cudaEventRecord(ev_done, cs), "event record");
  FFWD_CUDA(cudaStreamWaitEvent(s, ev_done, 0), "stream wait");
  return FFWD_OK;
}

int ffwd_rmsnorm(float* x, const float* gain, int T, int d, double eps, const void* add,
                 int add_kind, void* out_bf16, float* out_f32, const float* query, float* logits,
                 int logit_row0, int logit_row1, void* stream) {
  return ffwd_rmsnorm_ex(x, gain, T, d, eps, add, add_kind, out_bf16, out_f32, query, logits,
                         logit_row0, logit_row1, 0, stream);
}

int ffwd_rmsnorm_ex(float* x, const float* gain, int T, int d, double eps, const void* add,
                    int add_kind, void* out_bf16, float* out_f32, const float* query,
                    float* logits, int logit_row0, int logit_row1, int flags, void* stream) {
  g_err.clear();
  if (!x || !gain) return fail(FFWD_ERR_VALIDATION, "rmsnorm needs x and gain");
  if (flags & ~FFWD_NORM_LOGITS_F32) return fail(FFWD_ERR_VALIDATION, "unknown rmsnorm flags %d", flags);
  if ((flags & FFWD_NORM_LOGITS_F32) && query && !out_f32)
    return fail(FFWD_ERR_VALIDATION, "f32 logits need the f32 output the predictor pools");
  if (T < 1 || d < 4 || d % 4 != 0)
    return fail(FFWD_ERR_VALIDATION, "rmsnorm dims T=%d d=%d (d must be a positive multiple of 4)",
                T, d);
  if (d > 16384) return fail(FFWD_ERR_UNSUPPORTED, "rmsnorm supports d_model <= 16384, got %d", d);
  if (!out_bf16 && !out_f32) return fail(FFWD_ERR_VALIDATION, "rmsnorm needs an output");
  if (add && (add_kind < 1 || add_kind > 2))
    return fail(FFWD_ERR_VALIDATION, "rmsnorm add_kind must be 1 (f32) or 2 (bf16)");
  if (query && (!logits || logit_row0 < 0 || logit_row1 > T || logit_row0 > logit_row1))
    return fail(FFWD_ERR_VALIDATION, "rmsnorm logit rows [%d, %d) outside [0, %d)", logit_row0,
                logit_row1, T);
  const float sqrt_d = static_cast<float>(std::sqrt(static_cast<double>(d)));  // predictor.py:76
  StageTimer tm(kNorm, static_cast<cudaStream_t>(stream));
  FFWD_CUDA(launch_rmsnorm(x, gain, T, d, eps, add, add ? add_kind : 0, out_bf16, out_f32, query,
                           sqrt_d, logits, logit_row0, logit_row1,
                           (flags & FFWD_NORM_LOGITS_F32) != 0, static_cast<cudaStream_t>(stream)),
            "rmsnorm");
  return FFWD_OK;
}

int ffwd_rope(void* qk, int is_f32, int T, int row_stride, int k_col, int n_heads, int d_head,
              const double* cos_t, const double* sin_t, const float* cos32, const float* sin32,
              int pos0, void* stream) {
  g_err.clear();
  if (T < 1 || n_heads < 1 || d_head < 4 || d_head % 4 != 0)
    return fail(FFWD_ERR_VALIDATION, "rope dims T=%d heads=%d d_head=%d (d_head %% 4 == 0)", T,
                n_heads, d_head);
  if (k_col < n_heads * d_head || row_stride < k_col + n_heads * d_head)
    return fail(FFWD_ERR_VALIDATION, "rope layout: row_stride=%d k_col=%d for %d x %d", row_stride,
                k_col, n_heads, d_head);
  if (pos0 < 0) return fail(FFWD_ERR_VALIDATION, "rope pos0=%d < 0", pos0);
  if (!qk || !cos_t || !sin_t) return fail(FFWD_ERR_VALIDATION, "rope: null pointer");
  FFWD_CUDA(launch_rope(qk, is_f32 != 0, T, row_stride, k_col, n_heads, d_head, cos_t, sin_t,
                        cos32, sin32, pos0, static_cast<cudaStream_t>(stream)),
            "rope");
  return FFWD_OK;
}

int ffwd_timing_enable(int on) {
  g_timing = on != 0;
  return FFWD_OK;
}

int ffwd_timing_read(double* ms_out, int* count_out, int n_stages) {
  g_err.clear();
  for (int i = 0; i < n_stages; ++i) {
    if (ms_out) ms_out[i] = 0.0;
    if (count_out) count_out[i] = 0;
  }
  int rc = FFWD_OK;
  std::vector<Rec> recs;
  {
    std::lock_guard<std::mutex> lk(g_rec_mu);
    recs.swap(g_recs);
  }
  for (const Rec& r : recs) {
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e != cudaSuccess && rc == FFWD_OK) rc = cuda_fail(e, "timing_read");
    if (r.stage < n_stages) {
      if (ms_out) ms_out[r.stage] += ms;
      if (count_out) count_out[r.stage] += r.kernels;
    }
    std::lock_guard<std::mutex> lk(g_rec_mu);
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  return rc;
}

const char* ffwd_stage_name(int stage) {
  return (stage >= 0 && stage < kNumStages) ? kStageNames[stage] : "";
}

}  // extern "C"
