"""Per-layer neuron-activation predictor, run on the sm_100a pool/score kernels.

API mirrors the reference ``predictor.py:29-81``: ``default_reduced_dim``,
``PredictorParams``, ``init_predictor`` and ``predictor_forward``.  Scores are
accumulated in fp64 and rounded once to f32 exactly where the reference rounds,
so they are bit-identical to it (and the top-k indices derived from them exact).
The offline training routines (``predictor.py:84-171``) are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .errors import ValidationError
from .model import ModelConfig

F32 = np.float32


def default_reduced_dim(d_model: int) -> int:
    """Hidden width: d_model/16 rounded up to a power of two (``predictor.py:29-35``)."""
    r = 1
    while r < d_model / 16:
        r <<= 1
    return r


@dataclass
class PredictorParams:
    query: np.ndarray   # (1, d_model) pooling query
    w1: np.ndarray      # (d_model, r)
    w2: np.ndarray      # (r, d_ffn)

    @property
    def r(self) -> int:
        return self.w1.shape[1]

    def validate(self, cfg: ModelConfig) -> None:
        d, f = cfg.d_model, cfg.d_ffn
        if tuple(self.query.shape) != (1, d):
            raise ValidationError(f"predictor query shape {tuple(self.query.shape)}")
        if self.w1.shape[0] != d or tuple(self.w2.shape) != (self.w1.shape[1], f):
            raise ValidationError(
                f"predictor shapes inconsistent: w1 {tuple(self.w1.shape)}, "
                f"w2 {tuple(self.w2.shape)}")

    def on_device(self, device) -> "DevicePredictor":
        return DevicePredictor.from_params(self, device)


def init_predictor(cfg: ModelConfig, rng: np.random.Generator, r: int | None = None,
                   scale: float = 0.02) -> PredictorParams:
    """Gaussian init, draw order query, w1, w2 (``predictor.py:58-65``)."""
    r = default_reduced_dim(cfg.d_model) if r is None else r
    return PredictorParams(
        query=(rng.standard_normal((1, cfg.d_model)) * scale).astype(F32),
        w1=(rng.standard_normal((cfg.d_model, r)) * scale).astype(F32),
        w2=(rng.standard_normal((r, cfg.d_ffn)) * scale).astype(F32),
    )


@dataclass
class DevicePredictor:
    """f32 predictor parameters resident on the GPU (replicated under TP)."""
    query: torch.Tensor
    w1: torch.Tensor
    w2: torch.Tensor

    @property
    def d(self) -> int:
        return self.w1.shape[0]

    @property
    def r(self) -> int:
        return self.w1.shape[1]

    @property
    def f(self) -> int:
        return self.w2.shape[1]

    @classmethod
    def from_params(cls, p, device) -> "DevicePredictor":
        dev = torch.device(device)
        return cls(query=_dev.to_device(p.query, torch.float32, dev).reshape(-1),
                   w1=_dev.to_device(p.w1, torch.float32, dev),
                   w2=_dev.to_device(p.w2, torch.float32, dev))


def predictor_scores(dp: DevicePredictor, x: torch.Tensor, blk_begin: int = 0,
                     blk_count: int | None = None, block_size: int = 128) -> torch.Tensor:
    """Scores (blk_count, d_ffn) for 128-token blocks of a device tensor x (T, d)."""
    if block_size != 128:
        raise ValidationError("the sm_100a predictor kernels use 128-token blocks")
    if x.dim() != 2 or x.shape[1] != dp.d:
        raise ValidationError(f"predictor input shape {tuple(x.shape)}, d_model={dp.d}")
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.float()
    x = x.contiguous()
    T = x.shape[0]
    n_blk = -(-T // block_size)
    if blk_count is None:
        blk_count = n_blk - blk_begin
    lib = _dev.lib_for(x.device)
    scores = torch.empty((blk_count, dp.f), dtype=torch.float32, device=x.device)
    ws_n = lib.ffwd_predictor_workspace_bytes(blk_count, dp.d, dp.r, dp.f)
    ws = _dev.workspace(x.device, ws_n)
    _lib.check(lib.ffwd_predictor_forward(
        x.data_ptr(), int(x.dtype == torch.float32), T, dp.d, blk_begin, blk_count,
        dp.query.data_ptr(), dp.w1.data_ptr(), dp.w2.data_ptr(), dp.r, dp.f,
        scores.data_ptr(), ws.data_ptr(), ws.numel(), _dev.stream_handle(x.device)),
        "predictor_forward")
    return scores


def predictor_logits(dp: DevicePredictor, x: torch.Tensor) -> torch.Tensor:
    """Per-token logits f32(q . x_t) / f32(sqrt d) (``predictor.py:76``) of a device
    tensor x (T, d), f32 or bf16: the predictor's first pooling pass alone, in the f64
    order the fused RMSNorm producer shares (``ffwd_predictor_logits``)."""
    if x.dim() != 2 or x.shape[1] != dp.d:
        raise ValidationError(f"predictor input shape {tuple(x.shape)}, d_model={dp.d}")
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.float()
    x = x.contiguous()
    out = torch.empty((x.shape[0],), dtype=torch.float32, device=x.device)
    lib = _dev.lib_for(x.device)
    _lib.check(lib.ffwd_predictor_logits(x.data_ptr(), int(x.dtype == torch.float32), x.shape[0],
                                         dp.d, dp.query.data_ptr(), out.data_ptr(),
                                         _dev.stream_handle(x.device)), "predictor_logits")
    return out


def predictor_forward(params, x):
    """Neuron scores (d_ffn,) for one block of FFN inputs x (n, d_model).

    Drop-in for ``predictor.py:68-81``.  Pooling is non-causal over the whole
    block.  Accepts numpy (returns numpy f32) or CUDA tensors (returns a CUDA
    tensor); the arithmetic runs on the GPU either way.
    """
    host = _dev.is_host(x)
    d = params.w1.shape[0]
    shape = tuple(np.asarray(x).shape) if host else tuple(x.shape)
    if len(shape) != 2 or shape[1] != d or shape[0] < 1:
        raise ValidationError(f"predictor input shape {shape}, d_model={d}")
    dev = _dev.device_of(x, getattr(params, "w1", None))
    if isinstance(params, DevicePredictor):
        dp = params
    else:  # resident across calls (engine.py:286 calls this once per block and layer)
        key = (str(dev),) + _dev.fingerprint(params.query, params.w1, params.w2)
        dp = _dev.cached_on(params, "_ffwd_device", key,
                            lambda: DevicePredictor.from_params(params, dev))
    xt = _dev.to_device(x, torch.float32, dev) if host or x.dtype not in (
        torch.float32, torch.bfloat16) else x.contiguous()
    # one block of any n rows and any width (the reference pools whatever it is handed)
    lib = _dev.lib_for(dev)
    s = torch.empty((dp.f,), dtype=torch.float32, device=dev)
    ws = _dev.workspace(dev, lib.ffwd_predictor_workspace_bytes(1, dp.d, dp.r, dp.f))
    _lib.check(lib.ffwd_predictor_forward_block(
        xt.data_ptr(), int(xt.dtype == torch.float32), xt.shape[0], dp.d, dp.query.data_ptr(),
        dp.w1.data_ptr(), dp.w2.data_ptr(), dp.r, dp.f, s.data_ptr(), ws.data_ptr(), ws.numel(),
        _dev.stream_handle(dev)), "predictor_forward")
    return _dev.to_host_f32(s) if host else s
