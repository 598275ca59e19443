"""Expert masks, top-k selection and the gathered SwiGLU FFN (reference ``sparse.py``).

Same names and semantics as the reference (``sparse.py:18-91``,
``kernels.py:139-149``).  The one deliberate difference: ``SubWeights`` is a
lazy view (layer weights + index set) instead of three materialised copies
(``sparse.py:66-78``), because on the GPU the selected rows are gathered by
TMA straight from neuron-major weights inside the GEMM.  Accessing
``sub.w_gate`` / ``w_up`` / ``w_down`` still materialises the reference's
slices on the host for callers that want them.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .errors import ValidationError
from .model import LayerWeights


@dataclass
class ExpertMask:
    bits: np.ndarray          # (d_ffn,) uint8, exactly k ones
    k: int
    layer: int = -1
    block: int = -1
    indices: np.ndarray = field(init=False)

    def __post_init__(self):
        self.bits = np.asarray(self.bits, dtype=np.uint8)
        if self.bits.ndim != 1:
            raise ValidationError(f"mask bits must be 1-D, got {self.bits.shape}")
        if not np.isin(self.bits, (0, 1)).all():
            raise ValidationError("mask bits must be 0/1")
        pop = int(self.bits.sum())
        if pop != self.k:
            raise ValidationError(f"mask popcount {pop} != k={self.k}")
        self.indices = np.flatnonzero(self.bits).astype(np.int64)


def budget_to_k(b: float, d_ffn: int) -> int:
    """Neuron count for a keep fraction: round half up, clamp to [1, d_ffn] (``sparse.py:38-46``)."""
    if not 0.0 < b <= 1.0:
        raise ValidationError(f"keep fraction must be in (0, 1], got {b}")
    return min(d_ffn, max(1, int(np.floor(b * d_ffn + 0.5))))


def topk_device(scores: torch.Tensor, k: int) -> torch.Tensor:
    """Row-wise top-k of a CUDA (rows, f) f32 tensor -> ascending int32 (rows, k)."""
    if scores.dim() == 1:
        scores = scores.unsqueeze(0)
    scores = scores.to(torch.float32).contiguous()
    rows, f = scores.shape
    if not 1 <= k <= f:
        raise ValidationError(f"k={k} out of range [1, {f}]")
    lib = _dev.lib_for(scores.device)
    out = torch.empty((rows, k), dtype=torch.int32, device=scores.device)
    _lib.check(lib.ffwd_topk(scores.data_ptr(), rows, f, k, 0, 1, out.data_ptr(), k, None, 0,
                             None, _dev.stream_handle(scores.device)), "topk")
    return out


def topk_indices(scores, k: int):
    """Index set of the k largest scores; ties keep the lower index (``kernels.py:139-149``)."""
    host = _dev.is_host(scores)
    if host:
        s = np.asarray(scores, dtype=np.float32)
        if s.ndim != 1:
            raise ValidationError(f"scores must be 1-D, got shape {s.shape}")
        if not 1 <= k <= s.shape[0]:
            raise ValidationError(f"k={k} out of range [1, {s.shape[0]}]")
    elif scores.dim() != 1:
        raise ValidationError(f"scores must be 1-D, got shape {tuple(scores.shape)}")
    dev = _dev.device_of(scores)
    st = _dev.to_device(scores, torch.float32, dev)
    idx = topk_device(st, k)[0]
    return idx.cpu().numpy().astype(np.int64) if host else idx.to(torch.int64)


def build_mask(scores, k: int, layer: int = -1, block: int = -1) -> ExpertMask:
    """Top-k binary mask over neuron scores; ties keep the lower index (``sparse.py:49-55``)."""
    n = int(scores.shape[0]) if hasattr(scores, "shape") else len(scores)
    idx = topk_indices(scores, k)
    if isinstance(idx, torch.Tensor):
        idx = idx.cpu().numpy()
    bits = np.zeros(n, dtype=np.uint8)
    bits[idx] = 1
    return ExpertMask(bits=bits, k=k, layer=layer, block=block)


class SubWeights:
    """Lazy (weights, mask) view; replaces the materialised ``SubWeights`` (``sparse.py:58-63``)."""

    def __init__(self, lw: LayerWeights, mask: ExpertMask):
        self.lw = lw
        self.mask = mask

    @property
    def w_gate(self) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(self.lw.w_gate)[:, self.mask.indices])

    @property
    def w_up(self) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(self.lw.w_up)[:, self.mask.indices])

    @property
    def w_down(self) -> np.ndarray:
        return np.asarray(self.lw.w_down)[self.mask.indices]


def select_subweights(lw: LayerWeights, mask: ExpertMask) -> SubWeights:
    """Check the mask against the layer and return the lazy view (``sparse.py:66-78``)."""
    d_ffn = lw.w_gate.shape[1]
    if mask.bits.shape[0] != d_ffn:
        raise ValidationError(f"mask width {mask.bits.shape[0]} != d_ffn {d_ffn}")
    idx = mask.indices
    if idx.size == 0:
        raise ValidationError("row index set must not be empty")
    return SubWeights(lw, mask)


def sparse_ffn_forward(x, sub: SubWeights):
    """Gated FFN restricted to the selected neurons (``sparse.py:81-91``), on the GPU.

    silu(x . Wg[:, idx]) * (x . Wu[:, idx]) . Wd[idx, :] with bf16 operands and
    f32 accumulation (tolerance stated in DESIGN.md).
    """
    from .layer import packed_for, run_sparse_ffn
    host = _dev.is_host(x)
    dev = _dev.device_of(x)
    packed = packed_for(sub.lw, None, dev)
    idx = sub.mask.indices
    k = int(idx.size)
    ld = -(-k // 4) * 4
    row = np.zeros((1, ld), np.int32)
    row[0, :k] = idx
    idx_t = torch.from_numpy(row).to(dev)
    y = run_sparse_ffn(x, packed, idx_t, k=k, has_comp=False, idx_per_block=False)
    return _dev.to_host_f32(y) if host else y
