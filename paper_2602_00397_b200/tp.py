"""Tensor parallelism over d_ffn.

Rank s of N holds the neurons {j : j % N == s} (strided, so planted
contiguous neuron groups spread evenly) of W_gate / W_up / W_down and a
contiguous 1/N slice of the compensator bottleneck.  The predictor is
replicated: every rank computes the same global top-k (bit-exact, so no
collective is needed before the FFN) and keeps its local subset.  Each rank's
down projection yields a partial Y; one all-reduce (sum) per layer completes
it.  Independent prompts are data parallel and need no collective at all.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .compensator import CompensatorParams
from .errors import ValidationError
from .layer import PackedLayer, pack_layer, shard_comp_cols, shard_neurons, sparse_ffn_layer
from .predictor import DevicePredictor


def shard_host(w_gate, w_up, w_down, comp: CompensatorParams | None, tp_rank: int,
               tp_size: int):
    """Host-side (numpy) shard of one layer for rank `tp_rank`: the exact slices
    ``pack_layer`` uploads.  Returns (w_gate_s, w_up_s, w_down_s, comp_s, neuron_ids)."""
    f = np.asarray(w_gate).shape[1]
    nid = shard_neurons(f, tp_rank, tp_size)
    comp_s = None
    if comp is not None:
        lo, hi = shard_comp_cols(comp.w1.shape[1], tp_rank, tp_size)
        comp_s = CompensatorParams(w1=np.asarray(comp.w1)[:, lo:hi], w2=np.asarray(comp.w2)[lo:hi])
    return (np.asarray(w_gate)[:, nid], np.asarray(w_up)[:, nid], np.asarray(w_down)[nid],
            comp_s, nid)


def local_selection(global_idx: np.ndarray, tp_rank: int, tp_size: int) -> np.ndarray:
    """Rank-local ids (j // N) of the globally selected neurons this rank owns;
    the GPU top-k emits exactly this list (``ffwd_topk`` with tp_size > 1)."""
    g = np.asarray(global_idx)
    return g[g % tp_size == tp_rank] // tp_size


def allreduce_partial(y: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank partial FFN outputs in place (one collective per layer)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
    return y


@dataclass
class TensorParallelFFN:
    """One layer's FFN hot path on this rank: local sparse FFN + all-reduce."""
    packed: PackedLayer
    predictor: DevicePredictor
    k: int
    dense_first_last: bool = True
    group: object = None

    @classmethod
    def build(cls, w_gate, w_up, w_down, comp, predictor_params, k: int, device,
              tp_rank: int | None = None, tp_size: int | None = None,
              dense_first_last: bool = True, group=None) -> "TensorParallelFFN":
        if tp_size is None:
            tp_size = dist.get_world_size(group) if dist.is_initialized() else 1
        if tp_rank is None:
            tp_rank = dist.get_rank(group) if dist.is_initialized() else 0
        if not 0 <= tp_rank < tp_size:
            raise ValidationError(f"bad tensor-parallel rank {tp_rank} of {tp_size}")
        packed = pack_layer(w_gate, w_up, w_down, comp, device=device, tp_rank=tp_rank,
                            tp_size=tp_size)
        dp = DevicePredictor.from_params(predictor_params, device)
        return cls(packed, dp, k, dense_first_last, group)

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        y = sparse_ffn_layer(x, self.packed, self.predictor, self.k,
                             dense_first_last=self.dense_first_last, out=out)
        return allreduce_partial(y, self.group)
