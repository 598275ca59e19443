"""CPU oracle for the FastForward prefill-FFN hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2602_00397_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, and only as the checker
or as the timed CPU baseline.  The product path runs on the sm_100a kernels
and fails loudly when they are missing.

This is a NumPy restatement of the reference algorithm
(``/root/reference/pkg/src/sparseprefill``), written from its documented
semantics; every function cites the reference file:line it restates.  It is
pinned against golden vectors produced by running the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``; checked by
``tests/test_oracle_golden.py``).

Numeric conventions restated from ``kernels.py:1-15``:
  * storage is float32; every matrix product accumulates in float64 and is
    rounded once to float32 (``kernels.py:41-54``);
  * softmax and SiLU evaluate in float64 and round to float32
    (``kernels.py:57-89``);
  * top-k is a stable descending sort: ties keep the lower index, NaN sorts
    after every number, and the kept set is returned ascending
    (``kernels.py:139-149``).
"""

from __future__ import annotations

import numpy as np

F32 = np.float32
F64 = np.float64


class OracleError(ValueError):
    """Raised for the same preconditions the reference rejects with ValidationError."""


# --------------------------------------------------------------------------- numerics
def mm(a, b) -> np.ndarray:
    """f32 x f32 -> f64 accumulate -> f32.  Restates ``kernels.py:41-54``."""
    a = np.asarray(a, dtype=F32)
    b = np.asarray(b, dtype=F32)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise OracleError(f"bad matmul shapes {a.shape} @ {b.shape}")
    return (a.astype(F64) @ b.astype(F64)).astype(F32)


def softmax_row(z) -> np.ndarray:
    """Non-causal row softmax in f64, rounded to f32.  ``kernels.py:57-80``."""
    z64 = np.asarray(z, dtype=F32).astype(F64)
    z64 = z64 - z64.max(axis=-1, keepdims=True)
    e = np.exp(z64)
    return (e / e.sum(axis=-1, keepdims=True)).astype(F32)


def silu(v) -> np.ndarray:
    """Overflow-safe x*sigmoid(x) in f64, rounded to f32.  ``kernels.py:83-89``."""
    x = np.asarray(v, dtype=F32).astype(F64)
    pos = x / (1.0 + np.exp(-np.abs(x)))
    with np.errstate(over="ignore", invalid="ignore"):
        ex = np.exp(x)
        neg = x * ex / (1.0 + ex)
    return np.where(x >= 0, pos, neg).astype(F32)


def relu(v) -> np.ndarray:
    """``kernels.py:92-93``."""
    return np.maximum(np.asarray(v, dtype=F32), F32(0.0))


def topk_indices(scores, k: int) -> np.ndarray:
    """Ascending index set of the k largest scores.  ``kernels.py:139-149``.

    Stable descending order: equal scores keep index order (so -0.0 and +0.0
    tie), NaN ranks below every number (NumPy sorts NaN last).
    """
    s = np.asarray(scores, dtype=F32)
    if s.ndim != 1:
        raise OracleError(f"scores must be 1-D, got {s.shape}")
    if not 1 <= k <= s.shape[0]:
        raise OracleError(f"k={k} out of range [1, {s.shape[0]}]")
    order = np.argsort(-s, kind="stable")
    return np.sort(order[:k]).astype(np.int64)


def budget_to_k(b: float, d_ffn: int) -> int:
    """Round-half-up neuron count, clamped to [1, d_ffn].  ``sparse.py:38-46``."""
    if not 0.0 < b <= 1.0:
        raise OracleError(f"keep fraction must be in (0, 1], got {b}")
    return min(d_ffn, max(1, int(np.floor(b * d_ffn + 0.5))))


def bf16_round(a) -> np.ndarray:
    """Round f32 values to the nearest bf16 (ties to even), returned as f32.

    Used by the parity protocol: both sides see the same
    bf16-representable weights and inputs.  NaN stays NaN.
    """
    a = np.ascontiguousarray(a, dtype=F32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    out = r.astype(np.uint32).view(F32).copy()
    nan = np.isnan(a)
    out[nan] = a[nan]
    return out


# --------------------------------------------------------------------------- shapes / init
def default_reduced_dim(d_model: int) -> int:
    """Predictor width: smallest power of two >= d/16.  ``predictor.py:29-35``."""
    r = 1
    while r < d_model / 16:
        r *= 2
    return r


def default_comp_dim(d_model: int) -> int:
    """Compensator width d//8, at least 1.  ``compensator.py:20-22``."""
    return max(1, d_model // 8)


def gaussian(rng: np.random.Generator, shape, scale: float) -> np.ndarray:
    return (rng.standard_normal(shape) * scale).astype(F32)


def random_layer(rng: np.random.Generator, d: int, f: int, scale: float = 0.02) -> dict:
    """Same draw order as ``synthetic.py:33-43``: wq, wk, wv, wo, gate, up, down."""
    out = {}
    for name, shape in (("wq", (d, d)), ("wk", (d, d)), ("wv", (d, d)), ("wo", (d, d)),
                        ("w_gate", (d, f)), ("w_up", (d, f)), ("w_down", (f, d))):
        out[name] = gaussian(rng, shape, scale)
    return out


def synthetic_model(seed: int, n_layers: int, d: int, f: int, vocab: int,
                    scale: float = 0.02, tied_output: bool = False) -> dict:
    """``synthetic.generate_synthetic_model`` (synthetic.py:46-61): one generator, draw
    order tok_emb, then every layer's random_layer, then the untied head; norm
    gains are ones."""
    rng = np.random.default_rng(seed)
    tok_emb = gaussian(rng, (vocab, d), scale)
    layers = []
    for _ in range(n_layers):
        lw = random_layer(rng, d, f, scale)
        lw["attn_norm"] = np.ones(d, F32)
        lw["ffn_norm"] = np.ones(d, F32)
        layers.append(lw)
    w_out = None if tied_output else gaussian(rng, (d, vocab), scale)
    return {"tok_emb": tok_emb, "layers": layers, "final_norm": np.ones(d, F32), "w_out": w_out}


def init_predictor(rng: np.random.Generator, d: int, f: int, r: int | None = None,
                   scale: float = 0.02) -> dict:
    """Draw order query, w1, w2.  ``predictor.py:58-65``."""
    r = default_reduced_dim(d) if r is None else r
    return {"query": gaussian(rng, (1, d), scale),
            "w1": gaussian(rng, (d, r), scale),
            "w2": gaussian(rng, (r, f), scale)}


def init_compensator(rng: np.random.Generator, d: int, r: int | None = None,
                     scale: float = 0.02) -> dict:
    """Draw order w1, w2.  ``compensator.py:42-49``."""
    r = default_comp_dim(d) if r is None else r
    return {"w1": gaussian(rng, (d, r), scale), "w2": gaussian(rng, (r, d), scale)}


# --------------------------------------------------------------------------- hot path
def predictor_forward(query, w1, w2, x) -> np.ndarray:
    """Scores (f,) for one block x (n, d).  ``predictor.py:68-81``.

    logits = f32(q.x^T) / f32(sqrt(d))  (true f32 division, ``:76``), softmax
    (``:77``), pooled = p.x (``:78``), relu(pooled.W1) (``:79``), .W2 (``:80``).
    """
    x = np.asarray(x, dtype=F32)
    d = query.shape[1]
    if x.ndim != 2 or x.shape[1] != d:
        raise OracleError(f"predictor input shape {x.shape}, d_model={d}")
    z = mm(query, x.T) / F32(np.sqrt(d))
    p = softmax_row(z)
    pooled = mm(p, x)
    h = relu(mm(pooled, w1))
    return mm(h, w2)[0]


def sparse_ffn_forward(x, w_gate, w_up, w_down, idx) -> np.ndarray:
    """Gated FFN over the selected neurons, with the reference's materialised
    sub-weight copies.  ``sparse.py:66-91`` (+ ``kernels.py:125-136``)."""
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size == 0 or (np.diff(idx) <= 0).any() or idx[0] < 0 or idx[-1] >= w_gate.shape[1]:
        raise OracleError("index set must be non-empty, strictly increasing, in range")
    g_sub = np.ascontiguousarray(w_gate[:, idx])
    u_sub = np.ascontiguousarray(w_up[:, idx])
    d_sub = w_down[idx]
    hidden = silu(mm(x, g_sub)) * mm(x, u_sub)
    return mm(hidden, d_sub)


def dense_ffn(x, w_gate, w_up, w_down) -> np.ndarray:
    """``engine.py:127-131``."""
    return mm(silu(mm(x, w_gate)) * mm(x, w_up), w_down)


def compensator_forward(w1, w2, x) -> np.ndarray:
    """silu(x.W1).W2.  ``compensator.py:52-58``."""
    return mm(silu(mm(x, w1)), w2)


def block_spans(T: int, block: int) -> list[tuple[int, int]]:
    """Block partition with a short tail.  ``engine.py:254-257``, ``model.py:67-68``."""
    return [(lo, min(T, lo + block)) for lo in range(0, T, block)]


def ffn_layer_blockwise(x, lw: dict, pred: dict | None, comp: dict | None, k: int,
                        dense_first_last: bool = True, block: int = 128,
                        keep_masks: bool = False):
    """The FFN branch of ``prefill_blockwise`` for one layer, all blocks.

    Restates ``engine.py:254-310`` (mode="predicted"): dense FFN on the first
    and last block when ``dense_first_last`` (``:258-262``) or when k == d_ffn
    (``:268-279``); otherwise predictor -> top-k -> gathered sparse FFN
    (``:284-295``) and, if a compensator is given, + silu(x.Wc1).Wc2
    (``:296-300``).  Returns (y, {block: indices}, {block: scores}).
    """
    x = np.asarray(x, dtype=F32)
    T, _ = x.shape
    f = lw["w_gate"].shape[1]
    spans = block_spans(T, block)
    y = np.empty_like(x)
    masks, scores_out = {}, {}
    for j, (lo, hi) in enumerate(spans):
        xb = x[lo:hi]
        dense = (dense_first_last and (j == 0 or j == len(spans) - 1)) or k == f
        if dense:
            y[lo:hi] = dense_ffn(xb, lw["w_gate"], lw["w_up"], lw["w_down"])
            continue
        s = predictor_forward(pred["query"], pred["w1"], pred["w2"], xb)
        idx = topk_indices(s, k)
        yb = sparse_ffn_forward(xb, lw["w_gate"], lw["w_up"], lw["w_down"], idx)
        if comp is not None:
            yb = yb + compensator_forward(comp["w1"], comp["w2"], xb)
        y[lo:hi] = yb
        if keep_masks:
            masks[j] = idx
            scores_out[j] = s
    return y, masks, scores_out


# --------------------------------------------------------------------------- scheduler
def allocate_budgets(s, budget: float) -> np.ndarray:
    """Algorithm 1: sequential capped proportional shares.  ``scheduler.py:66-93``."""
    s = np.asarray(s, dtype=F64)
    if s.ndim != 1 or s.size == 0:
        raise OracleError("importance scores must be a non-empty 1-D array")
    if not 0.0 < budget <= 1.0:
        raise OracleError(f"budget must be in (0, 1], got {budget}")
    if (s < 0).any():
        raise OracleError("importance scores must be non-negative")
    mass = float(s.sum())
    if mass <= 0.0:
        raise OracleError("importance scores sum to zero")
    pool = budget * s.size
    out = np.zeros_like(s)
    for i in range(s.size):
        share = max(0.0, min(1.0, float(s[i]) / mass * pool)) if mass > 0 else 0.0
        out[i] = share
        pool -= share
        mass -= float(s[i])
    return out


# --------------------------------------------------------------------------- FLOPs
def layer_flops(T: int, d: int, f: int, k: int, dense_first_last: bool = True,
                block: int = 128, r: int | None = None, rc: int | None = None,
                has_comp: bool = True) -> dict:
    """Per-layer FFN-side FLOPs of the predicted path.  ``costmodel.py:151-175``."""
    r = default_reduced_dim(d) if r is None else r
    rc = default_comp_dim(d) if rc is None else rc
    spans = block_spans(T, block)
    out = {"ffn": 0, "predictor": 0, "compensator": 0}
    for j, (lo, hi) in enumerate(spans):
        n = hi - lo
        if (dense_first_last and (j == 0 or j == len(spans) - 1)) or k == f:
            out["ffn"] += 6 * n * d * f
            continue
        out["predictor"] += 4 * n * d + 2 * d * r + 2 * r * f
        out["ffn"] += 6 * n * d * k
        if has_comp:
            out["compensator"] += 4 * n * d * rc
    return out
