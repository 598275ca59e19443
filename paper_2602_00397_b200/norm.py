"""FFN-input producers of the full prefill on the sm_100a kernels (``csrc/norm.cu``).

``rmsnorm`` is ``kernels.rmsnorm`` (``kernels.py:96-106``) on a device f32
residual stream, optionally fused with the predictor's per-token logits
(``predictor.py:76``); ``apply_rope`` is ``engine.apply_rope``
(``engine.py:50-68``) in place on the Q and K columns of a fused QKV buffer.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .errors import ValidationError
from .predictor import DevicePredictor

ROPE_BASE = 10000.0  # engine.py:41


def rmsnorm(x: torch.Tensor, gain: torch.Tensor, eps: float = 1e-6, out_bf16: bool = True,
            out_f32: bool = False, predictor: DevicePredictor | None = None,
            logits: torch.Tensor | None = None, out: torch.Tensor | None = None,
            out32: torch.Tensor | None = None, add: torch.Tensor | None = None,
            logits_from_f32: bool = False):
    """Rows of x (T, d) f32 scaled to unit RMS times `gain` (f64 arithmetic, f32 result).

    With `add` ((T, d) f32 or bf16) the residual add ``x += add`` runs first, in place.

    Returns (bf16 or None, f32 or None, logits or None).  With `predictor`, also
    writes f32(q . bf16(row)) / f32(sqrt d) per row into `logits` (T,), the input of
    the predictor's pooling pass (``sparse_ffn_layer(..., logits_in=...)``); with
    ``logits_from_f32`` the dot product takes the f32 row instead (needs ``out_f32``;
    the predictor then pools that f32 copy: ``sparse_ffn_layer(..., x_pred_f32=...)``,
    the reference's predictor input, ``engine.py:267,286``).  The f64 summation order
    is the predictor's own (``csrc/rowdot.cuh``), so fused logits equal unfused ones bit
    for bit.
    """
    if logits_from_f32 and predictor is not None and not out_f32:
        raise ValidationError("logits_from_f32 needs out_f32 (the predictor pools the f32 rows)")
    if not (x.is_cuda and x.dtype == torch.float32 and x.dim() == 2 and x.is_contiguous()):
        raise ValidationError("rmsnorm expects a contiguous CUDA f32 (T, d) tensor")
    T, d = x.shape
    dev = x.device
    g = gain if (isinstance(gain, torch.Tensor) and gain.is_cuda) else \
        _dev.to_device(gain, torch.float32, dev)
    if tuple(g.shape) != (d,):
        raise ValidationError(f"gain shape {tuple(g.shape)} does not match row width {d}")
    ob = None
    if out_bf16:
        ob = out if out is not None else torch.empty((T, d), dtype=torch.bfloat16, device=dev)
    o32 = None
    if out_f32:
        o32 = out32 if out32 is not None else torch.empty((T, d), dtype=torch.float32, device=dev)
    q = None
    if predictor is not None:
        q = predictor.query
        if logits is None:
            logits = torch.empty((T,), dtype=torch.float32, device=dev)
    add_kind = 0
    if add is not None:
        if not (add.is_cuda and add.is_contiguous() and tuple(add.shape) == (T, d)
                and add.dtype in (torch.float32, torch.bfloat16)):
            raise ValidationError("rmsnorm add must be a contiguous CUDA f32/bf16 (T, d) tensor")
        add_kind = 1 if add.dtype == torch.float32 else 2
    lib = _dev.lib_for(dev)
    _lib.check(lib.ffwd_rmsnorm_ex(x.data_ptr(), g.data_ptr(), T, d, float(eps), _dev.ptr(add),
                                   add_kind, _dev.ptr(ob), _dev.ptr(o32), _dev.ptr(q),
                                   _dev.ptr(logits if q is not None else None), 0,
                                   T if q is not None else 0,
                                   1 if (logits_from_f32 and q is not None) else 0,
                                   _dev.stream_handle(dev)), "rmsnorm")
    return ob, o32, (logits if q is not None else None)


_rope_cache: dict = {}


def rope_tables(n_pos: int, d_head: int, device) -> tuple:
    """cos/sin tables [n_pos x d_head/2] with the reference's formula (engine.py:59-62):
    (cos f64, sin f64, cos f32, sin f32)."""
    dev = torch.device(device)
    key = (str(dev), d_head)
    hit = _rope_cache.get(key)
    if hit is not None and hit[0].shape[0] >= n_pos:
        return hit
    half = d_head // 2
    freqs = ROPE_BASE ** (-2.0 * np.arange(half) / d_head)
    ang = np.arange(n_pos)[:, None].astype(np.float64) * freqs[None, :]
    c64, s64 = torch.from_numpy(np.cos(ang)).to(dev), torch.from_numpy(np.sin(ang)).to(dev)
    tabs = (c64, s64, c64.float(), s64.float())
    _rope_cache[key] = tabs
    return tabs


def apply_rope(qkv: torch.Tensor, n_heads: int, d_head: int, pos0: int = 0,
               k_col: int | None = None) -> torch.Tensor:
    """Rotate the Q (columns [0, d)) and K (columns [k_col, k_col + d)) heads in place."""
    if not (qkv.is_cuda and qkv.dim() == 2 and qkv.is_contiguous()
            and qkv.dtype in (torch.bfloat16, torch.float32)):
        raise ValidationError("apply_rope expects a contiguous CUDA bf16/f32 (T, cols) tensor")
    T, stride = qkv.shape
    d = n_heads * d_head
    kc = d if k_col is None else k_col
    cos_t, sin_t, cos32, sin32 = rope_tables(pos0 + T, d_head, qkv.device)
    is_f32 = qkv.dtype == torch.float32
    lib = _dev.lib_for(qkv.device)
    _lib.check(lib.ffwd_rope(qkv.data_ptr(), int(is_f32), T, stride, kc, n_heads, d_head,
                             cos_t.data_ptr(), sin_t.data_ptr(),
                             None if is_f32 else cos32.data_ptr(),
                             None if is_f32 else sin32.data_ptr(), pos0,
                             _dev.stream_handle(qkv.device)), "rope")
    return qkv
