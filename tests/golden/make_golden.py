"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``sparseprefill`` from /root/reference/pkg/src (read-only; nothing
is copied) and writes small ``.npz`` fixtures next to this script.  The
fixtures pin the CPU oracle (``oracle/ffwd_oracle.py``) and feed the GPU
parity tests; /root/reference is never read at test time.

Parity protocol: FFN and compensator weights and the block
inputs are rounded to bf16 and handed to the reference as f32; predictor
parameters stay f32.  Seeds follow the reference: layer weights from
``synthetic._random_layer`` on ``default_rng([seed, layer, 7])``, predictor
on ``default_rng([seed, layer])`` (training.py:101), compensator on
``default_rng([seed + 1, layer])`` (training.py:204), inputs on
``default_rng([seed, layer, 99])`` ~ N(0, 1).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(HERE, "..", ".."))

from sparseprefill import kernels as rk  # noqa: E402
from sparseprefill.compensator import (apply_compensation, compensator_forward,  # noqa: E402
                                       init_compensator)
from sparseprefill.engine import dense_ffn  # noqa: E402
from sparseprefill.model import ModelConfig  # noqa: E402
from sparseprefill.predictor import PredictorParams, init_predictor, predictor_forward  # noqa: E402
from sparseprefill.scheduler import allocate_budgets  # noqa: E402
from sparseprefill.sparse import (budget_to_k, build_mask, select_subweights,  # noqa: E402
                                  sparse_ffn_forward)
from sparseprefill.synthetic import _random_layer  # noqa: E402

from oracle.ffwd_oracle import bf16_round  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def make_case(name, d, f, T, seed=1234, layer=0, budget=0.5, dense_first_last=True,
              with_ffn=True, store_y_rows=None):
    cfg = ModelConfig(n_layers=1, d_model=d, d_ffn=f, n_heads=max(1, d // 64),
                      vocab_size=8, block_size=128, max_context=max(T, 128))
    pred = init_predictor(cfg, np.random.default_rng([seed, layer]))
    comp = init_compensator(cfg, np.random.default_rng([seed + 1, layer]))
    comp.w1 = bf16_round(comp.w1)
    comp.w2 = bf16_round(comp.w2)
    x = bf16_round(np.random.default_rng([seed, layer, 99]).standard_normal((T, d))
                   .astype(np.float32))
    k = budget_to_k(budget, f)
    lw = None
    if with_ffn:
        lw = _random_layer(np.random.default_rng([seed, layer, 7]), cfg, 0.02)
        lw.w_gate = bf16_round(lw.w_gate)
        lw.w_up = bf16_round(lw.w_up)
        lw.w_down = bf16_round(lw.w_down)
    n_blocks = cfg.n_blocks(T)
    y = np.zeros((T, d), np.float32)
    sparse_blocks, idx_list, score_list = [], [], []
    for j in range(n_blocks):
        lo, hi = j * 128, min(T, (j + 1) * 128)
        xb = x[lo:hi]
        dense = (dense_first_last and (j == 0 or j == n_blocks - 1)) or k == f
        if dense:
            if with_ffn:
                y[lo:hi] = dense_ffn(xb, lw)
            continue
        s = predictor_forward(pred, xb)
        mask = build_mask(s, k, layer=layer, block=j)
        sparse_blocks.append(j)
        idx_list.append(mask.indices.astype(np.int32))
        score_list.append(s.astype(np.float32))
        if with_ffn:
            yb = sparse_ffn_forward(xb, select_subweights(lw, mask))
            y[lo:hi] = apply_compensation(yb, compensator_forward(comp, xb))
    out = dict(d=d, f=f, T=T, k=k, seed=seed, layer=layer, budget=budget,
               dense_first_last=int(dense_first_last),
               sparse_blocks=np.array(sparse_blocks, np.int32),
               indices=np.stack(idx_list) if idx_list else np.zeros((0, k), np.int32),
               scores=np.stack(score_list) if score_list else np.zeros((0, f), np.float32),
               sha_x=sha(x), sha_pred=sha(pred.query, pred.w1, pred.w2),
               sha_comp=sha(comp.w1, comp.w2))
    if with_ffn:
        out["sha_ffn"] = sha(lw.w_gate, lw.w_up, lw.w_down)
        y64 = y.astype(np.float64)
        out["y_sum"] = y64.sum()
        out["y_sumsq"] = (y64 * y64).sum()
        if store_y_rows is None:
            out["y"] = y
        else:
            rows = np.array(store_y_rows, np.int64)
            out["y_rows"] = rows
            out["y"] = y[rows]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: d={d} f={f} T={T} k={k} sparse_blocks={sparse_blocks[:8]}")


def make_topk_edges():
    """Top-k semantics at the edges, answered by the reference's topk_indices."""
    cases = []
    rng = np.random.default_rng(5)
    raw = [
        (np.array([1.0, 3.0, 3.0, 3.0], np.float32), 2),
        (np.array([0.5, 0.7, 0.7, 0.5], np.float32), 3),
        (np.array([1.0, 1.0, 1.0, 1.0], np.float32), 2),
        (np.array([0.0, -0.0, 0.0, -0.0, 1e-45, -1e-45], np.float32), 3),
        (np.array([np.nan, 1.0, np.nan, -np.inf, np.inf, 0.0], np.float32), 4),
        (np.array([np.nan, 1.0, np.nan, -np.inf, np.inf, 0.0], np.float32), 6),
        (np.array([np.nan, np.nan, np.nan], np.float32), 2),
        (np.array([-np.inf, -np.inf, -1.0, np.inf], np.float32), 3),
        (np.array([0.9, 0.1, 0.5, 0.3], np.float32), 2),
        (np.array([0.2, 0.9, 0.4], np.float32), 3),
    ]
    for n in (1, 7, 33, 1000, 1376, 4097):
        for kind in ("normal", "ties", "quant"):
            if kind == "normal":
                s = rng.standard_normal(n).astype(np.float32)
            elif kind == "ties":
                s = rng.integers(-3, 4, n).astype(np.float32)
            else:
                s = (np.round(rng.standard_normal(n) * 8) / 8).astype(np.float32)
                s[rng.random(n) < 0.1] = -0.0
            for k in sorted({1, max(1, n // 2), n}):
                raw.append((s, k))
    packed_scores, packed_k, packed_idx, offs_s, offs_i = [], [], [], [0], [0]
    for s, k in raw:
        idx = rk.topk_indices(s, k)
        packed_scores.append(s)
        packed_idx.append(idx.astype(np.int32))
        packed_k.append(k)
        offs_s.append(offs_s[-1] + s.size)
        offs_i.append(offs_i[-1] + idx.size)
    np.savez_compressed(os.path.join(HERE, "topk_edges.npz"),
                        scores=np.concatenate(packed_scores), k=np.array(packed_k, np.int32),
                        indices=np.concatenate(packed_idx),
                        offs_s=np.array(offs_s, np.int64), offs_i=np.array(offs_i, np.int64))
    print(f"topk_edges: {len(raw)} cases")


def make_scheduler():
    rng = np.random.default_rng(9)
    S, B, OUT, BT = [], [], [], []
    fixed = [([4.0, 2.0, 1.0, 1.0], 0.5), ([1.0, 4.0], 0.9), ([1.0, 1.0, 100.0], 0.9),
             ([100.0, 1.0, 1.0], 0.9), ([3.7] * 6, 0.45), ([2.0, 2.0, 2.0], 1.0)]
    for s, b in fixed:
        S.append(np.array(s)); B.append(b)
    for _ in range(40):
        n = int(rng.integers(1, 40))
        s = rng.random(n) ** 3 + (0.0 if rng.random() < 0.5 else 0.05)
        if s.sum() == 0:
            continue
        S.append(s); B.append(float(rng.uniform(0.05, 1.0)))
    for s, b in zip(S, B):
        OUT.append(allocate_budgets(s, b))
    offs = np.cumsum([0] + [len(s) for s in S])
    ks_b = np.array([1.0, 0.5, 0.004, 0.25, 0.75, 0.3333, 1e-9, 0.49999], np.float64)
    ks_f = np.array([64, 7, 1376, 8192, 14336, 12288, 4096, 3])
    kk = np.array([[budget_to_k(float(b), int(f)) for f in ks_f] for b in ks_b], np.int64)
    np.savez_compressed(os.path.join(HERE, "scheduler.npz"), s=np.concatenate(S),
                        budget=np.array(B), b=np.concatenate(OUT), offs=offs,
                        k_budgets=ks_b, k_dffn=ks_f, k_out=kk)
    print(f"scheduler: {len(S)} allocations")


def make_prefill_case(name="prefill_small", seed=2026, n_layers=2, d=256, f=768, n_heads=4,
                      vocab=512, T=512, budget=0.5):
    """Full block-wise prefill (engine.prefill_blockwise, predicted mode, and
    prefill_dense) on a synthetic model; FFN and compensator weights bf16-rounded."""
    from sparseprefill.engine import prefill_blockwise, prefill_dense
    from sparseprefill.scheduler import uniform_plan
    from sparseprefill.synthetic import generate_synthetic_model
    cfg = ModelConfig(n_layers=n_layers, d_model=d, d_ffn=f, n_heads=n_heads, vocab_size=vocab,
                      block_size=128, max_context=T)
    w = generate_synthetic_model(cfg, seed)
    for lw in w.layers:
        lw.w_gate, lw.w_up, lw.w_down = (bf16_round(lw.w_gate), bf16_round(lw.w_up),
                                         bf16_round(lw.w_down))
    preds = [init_predictor(cfg, np.random.default_rng([seed, l])) for l in range(n_layers)]
    comps = []
    for l in range(n_layers):
        c = init_compensator(cfg, np.random.default_rng([seed + 1, l]))
        c.w1, c.w2 = bf16_round(c.w1), bf16_round(c.w2)
        comps.append(c)
    tokens = np.random.default_rng([seed, 5]).integers(0, vocab, T)
    plan = uniform_plan(n_layers, budget)
    res = prefill_blockwise(w, tokens, plan, mode="predicted", predictors=preds,
                            compensators=comps, keep_masks=True, compute_recall=True)
    dense = prefill_dense(w, tokens)
    extra = {}
    for mode in ("oracle", "static"):
        r = prefill_blockwise(w, tokens, plan, mode=mode, compensators=comps, keep_masks=True)
        mk = sorted(r.masks)
        extra[f"{mode}_mask_keys"] = np.array(mk, np.int32)
        extra[f"{mode}_masks"] = np.stack([r.masks[kk].indices.astype(np.int32) for kk in mk])
        extra[f"{mode}_hidden"] = r.hidden[::4].astype(np.float32)
        extra[f"{mode}_flops_total"] = np.int64(r.flops.total())
    keys = sorted(res.masks)
    out = dict(seed=seed, n_layers=n_layers, d=d, f=f, n_heads=n_heads, vocab=vocab, T=T,
               budget=budget, k=budget_to_k(budget, f),
               mask_keys=np.array(keys, np.int32),
               masks=np.stack([res.masks[kk].indices.astype(np.int32) for kk in keys]),
               hidden_rows=np.arange(0, T, 4), hidden=res.hidden[::4].astype(np.float32),
               last_logits=res.last_logits, dense_hidden=dense.hidden[::4].astype(np.float32),
               dense_last_logits=dense.last_logits,
               flops_total=np.int64(res.flops.total()),
               recall_per_layer=res.recall_per_layer, **extra,
               sha_model=sha(w.tok_emb, w.w_out, *[getattr(lw, n) for lw in w.layers for n in
                                                    ("wq", "wk", "wv", "wo", "w_gate", "w_up",
                                                     "w_down")]),
               sha_pred=sha(*[a for p in preds for a in (p.query, p.w1, p.w2)]),
               sha_comp=sha(*[a for c in comps for a in (c.w1, c.w2)]),
               sha_tokens=sha(tokens))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {len(keys)} masks, flops {res.flops.total()}")


def make_checkpoint_case(seed=77, n_layers=2, d=64, f=160, n_heads=2, vocab=50):
    """Small `.ffwd` files written by the reference's own writer (checkpoint.py:77-118):
    a model file and an auxiliary predictor + compensator file."""
    from sparseprefill.checkpoint import write_checkpoint
    from sparseprefill.synthetic import generate_synthetic_model
    cfg = ModelConfig(n_layers=n_layers, d_model=d, d_ffn=f, n_heads=n_heads, vocab_size=vocab,
                      block_size=128, max_context=256)
    w = generate_synthetic_model(cfg, seed)
    preds = [init_predictor(cfg, np.random.default_rng([seed, l])) for l in range(n_layers)]
    comps = [init_compensator(cfg, np.random.default_rng([seed + 1, l])) for l in range(n_layers)]
    write_checkpoint(os.path.join(HERE, "tiny_model.ffwd"), cfg, weights=w)
    write_checkpoint(os.path.join(HERE, "tiny_aux.ffwd"), cfg, predictors=preds,
                     compensators=comps)
    print("tiny_model.ffwd / tiny_aux.ffwd written")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "prefill":
        make_prefill_case()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "checkpoint":
        make_checkpoint_case()
        sys.exit(0)
    make_topk_edges()
    make_scheduler()
    # tiny, with a short final block (300 = 128 + 128 + 44)
    make_case("tiny_dfl", d=128, f=384, T=300, seed=11, dense_first_last=True)
    make_case("tiny_all", d=128, f=384, T=300, seed=12, dense_first_last=False)
    make_case("tiny_k25", d=256, f=704, T=512, seed=13, budget=0.25, dense_first_last=False)
    # BASELINE configs[0] (the CPU reference case): d512 f1376 T1024, 50%
    make_case("cfg1", d=512, f=1376, T=1024, seed=2026, store_y_rows=list(range(120, 140))
              + list(range(500, 520)) + list(range(1000, 1024)))
    # Llama-3.2-1B shape, 4 blocks, outputs sampled
    make_case("l1b", d=2048, f=8192, T=512, seed=7, store_y_rows=list(range(128, 160))
              + list(range(300, 310)))
    # Llama-3.1-8B and Qwen3-8B shapes: predictor + top-k only (scores do not
    # depend on the FFN weights)
    make_case("l8b_pred", d=4096, f=14336, T=512, seed=8, with_ffn=False,
              dense_first_last=False)
    make_case("qwen8b_pred", d=4096, f=12288, T=384, seed=9, with_ffn=False,
              dense_first_last=False, budget=0.37)
    make_prefill_case()
    make_checkpoint_case()
