"""Full prefill on the GPU: the TTFT path around the FFN hot path.

Mirrors ``engine.prefill_blockwise`` / ``engine.prefill_dense``
(``engine.py:160-320``) for the ``dense`` and ``predicted`` modes, run
layer-major over the whole prompt (every attention is causal, so a block's
result depends only on earlier tokens; SURVEY 3.1 checks the equivalence):

    h = tok_emb[tokens]                                        engine.py:140-157
    per layer l:
        a   = rmsnorm(h, attn_norm)          ffwd_rmsnorm        engine.py:264
        qkv = a @ [Wq | Wk | Wv]             cuBLAS (library GEMM)  engine.py:86-88
        q,k = rope(q, k)                     ffwd_rope           engine.py:91-92
        o   = causal softmax(q k^T / sqrt(dh)) v   torch SDPA (cuDNN / flash)
        h  += o @ Wo                         cuBLAS              engine.py:107
        x   = rmsnorm(h, ffn_norm)           ffwd_rmsnorm + predictor logits
        h  += FFN(x)                         sparse_ffn_layer (predictor, top-k,
                                             gather-GEMMs, compensator, residual)
    logits = rmsnorm(h[-1], final_norm) @ head                engine.py:160-166

Attention is not the hot path: its GEMMs and the softmax go to
cuBLAS and PyTorch's SDPA.  ``attn_dtype=torch.float32`` runs the whole
attention side in f32 (and feeds the predictor the f32 RMSNorm output), which
is the parity mode the tests compare with the reference engine.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

from . import _dev
from .compensator import CompensatorParams
from .costmodel import FlopsReport, predict_prefill_flops
from .errors import ValidationError
from .layer import BLOCK, PackedLayer, ffn_layer_mode, oracle_scores, pack_layer, sparse_ffn_layer
from .model import ModelConfig
from .norm import apply_rope, rmsnorm
from .predictor import DevicePredictor, PredictorParams
from .sparse import budget_to_k, topk_device

MODES = ("dense", "oracle", "predicted", "static")
FUSE_LOGITS = True  # predictor logits from the FFN-input RMSNorm (A/B knob)
# Library attention backends, best first on sm_100 (cuDNN has Blackwell kernels).
SDPA_BACKENDS = [SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION,
                 SDPBackend.EFFICIENT_ATTENTION, SDPBackend.MATH]


@dataclass
class DeviceLayer:
    wqkv_t: torch.Tensor        # [3d x d]: (x @ [Wq|Wk|Wv])^T operand, attn dtype
    wo_t: torch.Tensor          # [d x d]: Wo^T, attn dtype
    attn_norm: torch.Tensor     # f32 (d,)
    ffn_norm: torch.Tensor      # f32 (d,)
    ffn: PackedLayer
    predictor: DevicePredictor | None
    k: int                      # neurons kept on predicted blocks (k == d_ffn: dense)


@dataclass
class DeviceModel:
    config: ModelConfig
    tok_emb: torch.Tensor       # f32 (V, d)
    layers: list
    final_norm: torch.Tensor    # f32 (d,)
    head: torch.Tensor          # f32 (d, V)
    dense_first_last: bool
    attn_dtype: torch.dtype
    has_comp: bool

    @classmethod
    def from_weights(cls, weights, plan=None, predictors=None, compensators=None,
                     device=None, attn_dtype: torch.dtype = torch.bfloat16) -> "DeviceModel":
        """Upload reference-layout weights (``ModelWeights``: ``x @ W`` orientation).

        ``plan`` (``SparsityPlan``) gives per-layer keep fractions and the
        dense-first/last flag; None = dense.  Predictors are required for layers
        with k < d_ffn (``engine.py:227-233``); compensators are optional.
        """
        cfg = weights.config
        if hasattr(weights, "validate"):
            weights.validate()
        dev = torch.device(device) if device is not None else _dev.device_of()
        L, d, f = cfg.n_layers, cfg.d_model, cfg.d_ffn
        if plan is not None:
            if len(plan.b) != L:
                raise ValidationError(f"plan has {len(plan.b)} budgets for {L} layers")
            ks = [budget_to_k(float(b), f) for b in plan.b]
            dfl = bool(plan.dense_first_last)
        else:
            ks, dfl = [f] * L, False
        if any(k < f for k in ks) and (predictors is None or len(predictors) != L):
            raise ValidationError("predicted mode requires one predictor per layer")
        if compensators is not None and len(compensators) != L:
            raise ValidationError("need one compensator per layer")

        def up(a, dt):
            return _dev.to_device(a, dt, dev)

        layers = []
        for l, lw in enumerate(weights.layers):
            wqkv = np.concatenate([np.asarray(lw.wq), np.asarray(lw.wk), np.asarray(lw.wv)],
                                  axis=1)
            comp = None
            if compensators is not None:
                c = compensators[l]
                comp = c if isinstance(c, CompensatorParams) else CompensatorParams(**c)
            pred = None
            if predictors is not None:
                p = predictors[l]
                pred = DevicePredictor.from_params(
                    p if isinstance(p, PredictorParams) else PredictorParams(**p), dev)
            layers.append(DeviceLayer(
                wqkv_t=up(wqkv.T, attn_dtype), wo_t=up(np.asarray(lw.wo).T, attn_dtype),
                attn_norm=up(lw.attn_norm, torch.float32), ffn_norm=up(lw.ffn_norm, torch.float32),
                ffn=pack_layer(lw.w_gate, lw.w_up, lw.w_down, comp, device=dev),
                predictor=pred, k=ks[l]))
        head = weights.out_head() if hasattr(weights, "out_head") else weights.w_out
        return cls(config=cfg, tok_emb=up(weights.tok_emb, torch.float32), layers=layers,
                   final_norm=up(weights.final_norm, torch.float32),
                   head=up(head, torch.float32), dense_first_last=dfl, attn_dtype=attn_dtype,
                   has_comp=compensators is not None)


@dataclass
class PrefillResult:
    hidden: torch.Tensor            # (T, d) f32 final-layer residual stream
    last_logits: torch.Tensor       # (V,) f32
    flops: FlopsReport
    masks: dict | None = None       # (layer, block) -> int64 ascending neuron ids
    kv: list | None = None          # per layer (rotated K, V), each (T, d)
    recall_per_layer: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


_dummy: dict = {}


def _dense_predictor(d: int, f: int, dev) -> DevicePredictor:
    key = (d, f, str(dev))
    if key not in _dummy:  # shape carrier only: k == d_ffn never runs the predictor
        z = torch.zeros
        _dummy[key] = DevicePredictor(query=z(d, device=dev), w1=z((d, 1), device=dev),
                                      w2=z((1, f), device=dev))
    return _dummy[key]


def _embed(model: DeviceModel, tokens) -> torch.Tensor:
    cfg = model.config
    ids = torch.as_tensor(np.asarray(tokens) if not isinstance(tokens, torch.Tensor) else tokens)
    if ids.dim() != 1 or ids.numel() == 0:
        raise ValidationError("token sequence must be a non-empty 1-D array")
    if ids.dtype.is_floating_point or ids.dtype == torch.bool:
        raise ValidationError(f"token ids must be integers, got {ids.dtype}")
    if ids.numel() > cfg.max_context:
        raise ValidationError(f"sequence length {ids.numel()} exceeds "
                              f"max_context={cfg.max_context}")
    lo, hi = int(ids.min()), int(ids.max())
    if lo < 0 or hi >= cfg.vocab_size:
        raise ValidationError(f"token ids must lie in [0, {cfg.vocab_size}), got [{lo}, {hi}]")
    return model.tok_emb.index_select(0, ids.to(model.tok_emb.device, torch.long)).contiguous()


def _attention(model: DeviceModel, dl: DeviceLayer, a: torch.Tensor, T: int):
    cfg = model.config
    H, dh, d = cfg.n_heads, cfg.d_head, cfg.d_model
    qkv = torch.mm(a, dl.wqkv_t.t())                       # (T, 3d)
    apply_rope(qkv, H, dh, pos0=0, k_col=d)
    q = qkv[:, :d].view(T, H, dh).transpose(0, 1).unsqueeze(0)
    k = qkv[:, d:2 * d].view(T, H, dh).transpose(0, 1).unsqueeze(0)
    v = qkv[:, 2 * d:].view(T, H, dh).transpose(0, 1).unsqueeze(0)
    with sdpa_kernel(SDPA_BACKENDS, set_priority=True):
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True)  # scale 1/sqrt(dh)
    o = o.squeeze(0).transpose(0, 1).reshape(T, d)
    return torch.mm(o, dl.wo_t.t()), qkv


def prefill(model: DeviceModel, tokens, mode: str = "predicted", keep_masks: bool = False,
            return_kv: bool = False, compute_recall: bool = False) -> PrefillResult:
    """Prefill `tokens` through every layer; returns the hidden states and last logits.

    Modes as ``engine.py:170-180``: ``dense``; ``predicted`` (the hot path); ``oracle``
    (each sparse block keeps the top-k of its own dense hidden norms); ``static`` (block
    0 dense, its masks reused by every later block).  ``compute_recall`` (predicted
    mode) measures each layer's mask recall against the oracle masks with an extra,
    uncounted dense scoring pass (``engine.py:192-199, 301-305``).
    """
    if mode not in MODES:
        raise ValidationError(f"unknown mode {mode!r}; expected one of {MODES}")
    cfg = model.config
    d, f = cfg.d_model, cfg.d_ffn
    h = _embed(model, tokens)                               # f32 (T, d) residual stream
    T = h.shape[0]
    dev = h.device
    f32_attn = model.attn_dtype == torch.float32
    n_blk = -(-T // BLOCK)
    masks = {} if keep_masks else None
    kv = [] if return_kv else None
    xb = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
    x32 = torch.empty((T, d), dtype=torch.float32, device=dev) if f32_attn else None
    lg = torch.empty((T,), dtype=torch.float32, device=dev)
    recall = np.full(cfg.n_layers, np.nan) if (compute_recall and mode == "predicted") else None
    for l, dl in enumerate(model.layers):
        a_bf, a32, _ = rmsnorm(h, dl.attn_norm, out_bf16=not f32_attn, out_f32=f32_attn)
        o, qkv = _attention(model, dl, a32 if f32_attn else a_bf, T)
        if return_kv:
            kv.append((qkv[:, d:2 * d].clone(), qkv[:, 2 * d:].clone()))
        k = f if mode == "dense" else dl.k
        sparse = k < f
        if mode in ("oracle", "static") and sparse:
            rmsnorm(h, dl.ffn_norm, out=xb, add=o)   # h += o (engine.py:265), x = norm(h)
            res = ffn_layer_mode(xb, dl.ffn, k, mode, dense_first_last=model.dense_first_last,
                                 has_comp=model.has_comp, out=h, residual=h,
                                 return_indices=keep_masks)
            if keep_masks:
                idx = res[1].cpu().numpy().astype(np.int64)
                if mode == "static":  # engine.py:273-277 and :306-307: one mask, every block
                    last = n_blk - 1 if model.dense_first_last else n_blk
                    for j in [0] + list(range(1, last)):
                        masks[(l, j)] = idx[0]
                else:
                    b0 = 1 if model.dense_first_last else 0
                    for row in range(idx.shape[0]):
                        masks[(l, b0 + row)] = idx[row]
            continue
        pred = dl.predictor if sparse else _dense_predictor(d, f, dev)
        fuse_logits = sparse and not f32_attn and FUSE_LOGITS
        # h += o (engine.py:265) fused into the FFN-input norm
        _, _, logits = rmsnorm(h, dl.ffn_norm, out=xb, out_f32=f32_attn and sparse, out32=x32,
                               predictor=pred if fuse_logits else None, logits=lg, add=o)
        want_idx = (keep_masks or recall is not None) and sparse
        if recall is not None and sparse:  # oracle masks of the same inputs (uncounted)
            osc = oracle_scores(xb, dl.ffn)
        res = sparse_ffn_layer(xb, dl.ffn, pred, k, dense_first_last=model.dense_first_last,
                               has_comp=model.has_comp, out=h, residual=h,
                               return_indices=want_idx,
                               x_pred_f32=x32 if (f32_attn and sparse) else None,
                               logits_in=logits if fuse_logits else None)
        if want_idx and res[1] is not None:  # None: no predicted block (short prompt)
            b0 = 1 if model.dense_first_last else 0
            idx = res[1]
            if recall is not None and idx.shape[0] > 0:
                oidx = topk_device(osc[b0:b0 + idx.shape[0]], k)
                inter = torch.stack([torch.isin(idx[r], oidx[r]).sum()
                                     for r in range(idx.shape[0])])
                recall[l] = float(inter.double().mean() / k)
            if keep_masks:
                idx = idx.cpu().numpy().astype(np.int64)
                for row in range(idx.shape[0]):
                    masks[(l, b0 + row)] = idx[row]
    fin = rmsnorm(h[-1:].contiguous(), model.final_norm, out_bf16=False, out_f32=True)[1]
    logits_out = torch.mv(model.head.t(), fin[0])  # f32 GEMV (the reference accumulates in f64)
    flops = predict_prefill_flops(
        cfg.n_layers, d, f, cfg.vocab_size, T, b=None if mode == "dense" else
        [float(dl.k) / f for dl in model.layers], dense_first_last=model.dense_first_last,
        mode=mode, has_compensators=model.has_comp)
    return PrefillResult(hidden=h, last_logits=logits_out, flops=flops, masks=masks, kv=kv,
                         recall_per_layer=recall, extra={"n_blocks": n_blk})
