"""Low-rank error compensator: API of the reference ``compensator.py:20-66``.

On the GPU the compensator is not a separate pass: its hidden layer
``silu(x . Wc1)`` is computed as extra N tiles of the up-projection kernel and
``. Wc2`` as extra K iterations of the down-projection kernel, accumulating
straight into the FFN output (``layer.sparse_ffn_layer``).  ``compensator_forward``
below runs that same machinery with an empty neuron set, so the correction
alone is available as a drop-in.  Training (``mse_distill_loss``) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from .errors import ValidationError
from .model import ModelConfig

F32 = np.float32


def default_comp_dim(d_model: int) -> int:
    """Bottleneck width d_model // 8, at least 1 (``compensator.py:20-22``)."""
    return max(1, d_model // 8)


@dataclass
class CompensatorParams:
    w1: np.ndarray   # (d_model, r_comp)
    w2: np.ndarray   # (r_comp, d_model)

    @property
    def r(self) -> int:
        return self.w1.shape[1]

    def validate(self, cfg: ModelConfig) -> None:
        d = cfg.d_model
        if self.w1.shape[0] != d or tuple(self.w2.shape) != (self.w1.shape[1], d):
            raise ValidationError(
                f"compensator shapes inconsistent: w1 {tuple(self.w1.shape)}, "
                f"w2 {tuple(self.w2.shape)}")


def init_compensator(cfg: ModelConfig, rng: np.random.Generator, r: int | None = None,
                     scale: float = 0.02) -> CompensatorParams:
    """Small Gaussian init, draw order w1, w2 (``compensator.py:42-49``)."""
    r = default_comp_dim(cfg.d_model) if r is None else r
    return CompensatorParams(
        w1=(rng.standard_normal((cfg.d_model, r)) * scale).astype(F32),
        w2=(rng.standard_normal((r, cfg.d_model)) * scale).astype(F32),
    )


def compensator_forward(params: CompensatorParams, x):
    """Correction term (n, d_model) for FFN inputs x (n, d_model), on the GPU.

    bf16 operands, f32 accumulation (tolerance in DESIGN.md).
    """
    from .layer import pack_layer, run_sparse_ffn  # local import: layer imports us
    d = params.w1.shape[0]
    xs = tuple(x.shape)
    if len(xs) != 2 or xs[1] != d:
        raise ValidationError(f"compensator input shape {xs}, d_model={d}")
    host = _dev.is_host(x)
    dev = _dev.device_of(x)

    def build():
        # an FFN with no neurons: one zero row stands in for the empty set
        zeros_in = torch.zeros((d, 1), dtype=torch.float32)
        zeros_out = torch.zeros((1, d), dtype=torch.float32)
        return (pack_layer(zeros_in, zeros_in, zeros_out, params, device=dev),
                torch.zeros((1, 4), dtype=torch.int32, device=dev))

    # packed once per params object and device, resident across calls (engine.py:296-300
    # calls this once per predicted block)
    key = (str(dev),) + _dev.fingerprint(params.w1, params.w2)
    packed, idx = _dev.cached_on(params, "_ffwd_packed", key, build)
    y = run_sparse_ffn(x, packed, idx, k=1, has_comp=True, idx_per_block=False)
    return _dev.to_host_f32(y) if host else y


def apply_compensation(y_sparse, correction):
    """``y + correction`` (``compensator.py:61-66``)."""
    if tuple(y_sparse.shape) != tuple(correction.shape):
        raise ValidationError(
            f"compensation shape mismatch: {tuple(y_sparse.shape)} vs {tuple(correction.shape)}")
    return y_sparse + correction
