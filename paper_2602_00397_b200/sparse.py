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


def hidden_column_scores(hidden):
    """Per-neuron L2 norm of gated activations across a block (``sparse.py:94-97``):
    f32(sqrt(sum_t h^2)) with f64 accumulation, on the GPU (``ffwd_column_norms``)."""
    host = _dev.is_host(hidden)
    dev = _dev.device_of(hidden)
    h = hidden if (not host and hidden.dtype in (torch.float32, torch.bfloat16)) else \
        _dev.to_device(hidden, torch.float32, dev)
    h = h.contiguous()
    if h.dim() != 2:
        raise ValidationError(f"hidden must be 2-D, got shape {tuple(h.shape)}")
    n, f = h.shape
    if n < 1:
        raise ValidationError("hidden must hold at least one row")
    out = torch.empty((1, f), dtype=torch.float32, device=dev)
    lib = _dev.lib_for(dev)
    _lib.check(lib.ffwd_column_norms(h.data_ptr(), int(h.dtype == torch.float32), n, f, f,
                                     out.data_ptr(), _dev.stream_handle(dev)), "column_norms")
    return out[0].cpu().numpy() if host else out[0]


def mask_from_hidden(hidden, k: int, layer: int = -1, block: int = -1) -> ExpertMask:
    """``sparse.py:100-102``: top-k of the hidden column norms."""
    return build_mask(hidden_column_scores(hidden), k, layer=layer, block=block)


def oracle_experts(x, lw: LayerWeights, k: int, layer: int = -1, block: int = -1) -> ExpertMask:
    """Exact top-k mask from a dense scoring pass over the block (``sparse.py:105-115``).

    The dense gate/up products run in the sm_100a up-projection (bf16 operands, f32
    accumulation, bf16 H), so scores near the k-th boundary may order differently
    from the reference's f32/f64 pass; this is an accuracy ceiling, not the hot path.
    """
    from .layer import oracle_scores, packed_for
    dev = _dev.device_of(x)
    packed = packed_for(lw, None, dev)
    s = oracle_scores(x, packed)
    if s.shape[0] != 1:
        raise ValidationError(f"one block of at most 128 tokens, got {s.shape[0]} blocks")
    return build_mask(s[0], k, layer=layer, block=block)


class FirstBlockStatic:
    """Reuse the first block's oracle masks for every later block (``sparse.py:118-137``)."""

    def __init__(self):
        self._masks: dict[int, ExpertMask] = {}

    def set_first(self, layer: int, mask: ExpertMask) -> None:
        self._masks[layer] = mask

    def mask_for(self, layer: int) -> ExpertMask:
        if layer not in self._masks:
            raise ValidationError(f"static mask requested for layer {layer} before the first "
                                  "block was processed")
        return self._masks[layer]
