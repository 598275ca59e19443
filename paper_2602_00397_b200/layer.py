"""Layer-batched FFN branch of the block-wise prefill on the sm_100a kernels.

``sparse_ffn_layer`` is the entry the engine would call once per layer
instead of the per-block loop of ``engine.py:254-310`` (FFN branch): by
layer-major equivalence every 128-token block of a layer is
handled in one stream-ordered sequence of launches:

    pool -> W1 -> W2 -> top-k  (K1, fp64-exact predictor, bit-exact indices)
    plan                       (device-side tile tables: no host sync)
    up-proj  (K2)              tcgen05 gather-GEMM, SiLU(g)*u epilogue, comp hidden
    down-proj (K3)             tcgen05 gather-GEMM, compensator as extra K

Weights are packed once per layer by ``pack_layer`` into the neuron-major
bf16 layout the kernels gather from (see include/ffwd_b200.h).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .compensator import CompensatorParams
from .errors import UnsupportedError, ValidationError
from .predictor import DevicePredictor

BLOCK = 128


def _rup(v: int, m: int) -> int:
    return -(-v // m) * m


def shard_neurons(f: int, tp_rank: int, tp_size: int) -> np.ndarray:
    """Global neuron ids held by a rank: strided {j : j % tp_size == tp_rank}."""
    if tp_size < 1 or not 0 <= tp_rank < tp_size:
        raise ValidationError(f"bad tensor-parallel rank {tp_rank} of {tp_size}")
    return np.arange(tp_rank, f, tp_size, dtype=np.int64)


def shard_comp_cols(rc: int, tp_rank: int, tp_size: int) -> tuple[int, int]:
    """Contiguous compensator-bottleneck columns [lo, hi) of a rank (np.array_split rule)."""
    base, extra = divmod(rc, tp_size)
    lo = tp_rank * base + min(tp_rank, extra)
    return lo, lo + base + (1 if tp_rank < extra else 0)


@dataclass
class PackedLayer:
    """One rank's FFN (+ compensator) weights in the kernels' neuron-major layout.

    ``d`` is the packed row width: d_model rounded up to 64 (the GEMMs' 128 B swizzle
    atom) with zero columns, which leave every product unchanged; ``d_model`` is the
    model's own width, to which inputs are padded and outputs sliced."""
    wgu_t: torch.Tensor   # bf16 [(2 f_local + roundup(rc_local, 256)) x d]
    wd: torch.Tensor      # bf16 [(f_local + roundup(rc_local, 64)) x d]
    d: int
    f_global: int
    f_local: int
    rc_local: int
    tp_rank: int = 0
    tp_size: int = 1
    d_model: int = 0

    def __post_init__(self):
        if not self.d_model:
            self.d_model = self.d

    @property
    def device(self) -> torch.device:
        return self.wgu_t.device


def _as_t(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32)))


def pack_layer(w_gate, w_up, w_down, comp: CompensatorParams | None = None, device=None,
               tp_rank: int = 0, tp_size: int = 1) -> PackedLayer:
    """Build the packed bf16 layout for one rank (one-time layout transform).

    w_gate/w_up (d, f) and w_down (f, d) in the reference orientation
    (``model.py:79-81``); comp.w1 (d, r'), comp.w2 (r', d) (``compensator.py:25-39``).
    """
    dev = torch.device(device) if device is not None else _dev.device_of()
    g, u, dn = _as_t(w_gate), _as_t(w_up), _as_t(w_down)
    d, f = g.shape
    if tuple(u.shape) != (d, f) or tuple(dn.shape) != (f, d):
        raise ValidationError(f"FFN weights inconsistent: gate {tuple(g.shape)}, "
                              f"up {tuple(u.shape)}, down {tuple(dn.shape)}")
    nid = torch.from_numpy(shard_neurons(f, tp_rank, tp_size))
    f_l = int(nid.numel())
    rc_l, c1, c2 = 0, None, None
    if comp is not None:
        c1, c2 = _as_t(comp.w1), _as_t(comp.w2)
        rc = c1.shape[1]
        if c1.shape[0] != d or tuple(c2.shape) != (rc, d):
            raise ValidationError("compensator shapes inconsistent with the FFN")
        lo, hi = shard_comp_cols(rc, tp_rank, tp_size)
        c1, c2 = c1[:, lo:hi], c2[lo:hi]
        rc_l = hi - lo
    bf = torch.bfloat16
    dp = _rup(d, 64)  # zero columns: the K2 contraction and K3's extra outputs ignore them
    nid_d = nid.to(dev) if g.is_cuda else nid
    wgu = torch.zeros((2 * f_l + _rup(rc_l, 256), dp), dtype=bf, device=dev)
    wgu[:f_l, :d] = g[:, nid_d].t().to(dev, bf)
    wgu[f_l:2 * f_l, :d] = u[:, nid_d].t().to(dev, bf)
    wd = torch.zeros((f_l + _rup(rc_l, 64), dp), dtype=bf, device=dev)
    wd[:f_l, :d] = dn[nid_d].to(dev, bf)
    if rc_l:
        wgu[2 * f_l:2 * f_l + rc_l, :d] = c1.t().to(dev, bf)
        wd[f_l:f_l + rc_l, :d] = c2.to(dev, bf)
    return PackedLayer(wgu_t=wgu, wd=wd, d=dp, f_global=f, f_local=f_l, rc_local=rc_l,
                       tp_rank=tp_rank, tp_size=tp_size, d_model=d)


def packed_for(lw, comp, device) -> PackedLayer:
    """Packed weights for reference-style layer weights, kept resident on the weights'
    own object (``_dev.cached_on``): the reference engine calls the drop-ins once per
    (block, layer) (``engine.py:263``), so a layer is packed once, not once per call.  The
    cache key is a fingerprint of the weight arrays (address, shape, torch version counter
    or a content sample), so replaced weights repack; see ``invalidate_packed``."""
    dev = torch.device(device)
    key = (str(dev),) + _dev.fingerprint(lw.w_gate, lw.w_up, lw.w_down,
                                         comp.w1 if comp is not None else None,
                                         comp.w2 if comp is not None else None)
    return _dev.cached_on(lw, "_ffwd_packed" if comp is None else "_ffwd_packed_comp", key,
                          lambda: pack_layer(lw.w_gate, lw.w_up, lw.w_down, comp, device=dev))


def invalidate_packed(obj) -> None:
    """Drop the device copies cached on a weights object (after editing it in place)."""
    store = getattr(obj, "__dict__", {})
    for slot in [k for k in store if k.startswith("_ffwd_")]:
        del store[slot]


def _x_bf16(x, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.bfloat16:
        return x.contiguous()
    return _dev.to_device(x, torch.bfloat16, dev)


def _pad_cols(xb: torch.Tensor, width: int) -> torch.Tensor:
    if xb.shape[1] == width:
        return xb
    out = torch.zeros((xb.shape[0], width), dtype=xb.dtype, device=xb.device)
    out[:, :xb.shape[1]] = xb
    return out


def run_sparse_ffn(x, packed: PackedLayer, idx: torch.Tensor | None, k: int,
                   has_comp: bool = False, idx_per_block: bool = True,
                   counts: torch.Tensor | None = None, out: torch.Tensor | None = None
                   ) -> torch.Tensor:
    """FFN over all 128-token blocks of x with given (rank-local) index rows.

    idx None -> dense FFN over every local neuron (``engine.py:127-131``).
    """
    dev = packed.device
    xb = _x_bf16(x, dev)
    if xb.dim() != 2 or xb.shape[1] != packed.d_model:
        raise ValidationError(f"FFN input shape {tuple(xb.shape)}, d_model={packed.d_model}")
    T = xb.shape[0]
    padded = packed.d != packed.d_model  # any d_model: zero columns up to the packed width
    xb = _pad_cols(xb, packed.d)
    lib = _dev.lib_for(dev)
    if padded:
        y = torch.empty((T, packed.d), dtype=torch.float32, device=dev)
    else:
        y = out if out is not None else torch.empty((T, packed.d), dtype=torch.float32,
                                                    device=dev)
    kk = packed.f_local if idx is None else k
    ws_n = lib.ffwd_sparse_ffn_workspace_bytes(T, packed.d, packed.f_local, packed.rc_local, kk)
    ws = _dev.workspace(dev, ws_n)
    ld = 0 if idx is None else idx.shape[1]
    _lib.check(lib.ffwd_sparse_ffn(
        xb.data_ptr(), T, packed.d, packed.wgu_t.data_ptr(), packed.wd.data_ptr(),
        packed.f_local, packed.rc_local, _dev.ptr(idx), int(idx_per_block), ld,
        _dev.ptr(counts), kk, int(has_comp and packed.rc_local > 0), y.data_ptr(),
        ws.data_ptr(), ws.numel(), _dev.stream_handle(dev)), "sparse_ffn")
    if padded:
        y = y[:, :packed.d_model]
        if out is not None:
            out.copy_(y)
            return out
        return y.contiguous()
    return y


def dense_ffn(x, packed: PackedLayer) -> torch.Tensor:
    """SiLU-gated FFN over all (local) neurons (``engine.py:127-131``), same kernels, identity index."""
    return run_sparse_ffn(x, packed, None, packed.f_local)


_DFL_CODES = {False: 0, True: 1, "first": 2, "last": 3}


def dense_first_last_code(v) -> int:
    """C-ABI code of ``dense_first_last``: a bool for a whole prompt (``engine.py:258-262``),
    or "first" / "last" for a sequence shard that holds only the prompt's first / last
    block (only that block runs dense)."""
    key = v if isinstance(v, str) else bool(v)
    if key not in _DFL_CODES:
        raise ValidationError(f"dense_first_last must be a bool, 'first' or 'last', got {v!r}")
    return _DFL_CODES[key]


def seq_shard(n_blk: int, rank: int, world: int):
    """Sequence parallelism over a prompt's 128-token blocks: rank ``rank`` of ``world``
    takes the contiguous blocks [b0, b1) and passes ``dense_first_last`` = the returned
    value, so only the ranks holding the prompt's first / last block run it dense
    (``engine.py:258-262``).  The FFN branch is block-local, so the shards need no
    collective."""
    if not 0 <= rank < world:
        raise ValidationError(f"bad sequence-parallel rank {rank} of {world}")
    if n_blk < world:
        raise ValidationError(f"{n_blk} blocks cannot feed {world} sequence-parallel ranks")
    b0, b1 = n_blk * rank // world, n_blk * (rank + 1) // world
    if world == 1:
        return b0, b1, True
    return b0, b1, "first" if rank == 0 else ("last" if rank == world - 1 else False)


def layer_workspace_bytes(T: int, packed: PackedLayer, r: int, k: int,
                          dense_first_last) -> int:
    lib = _dev.lib_for(packed.device)
    return int(lib.ffwd_layer_workspace_bytes(T, packed.d, packed.f_global, packed.f_local,
                                              packed.rc_local, r, k,
                                              dense_first_last_code(dense_first_last),
                                              packed.tp_size))


def sparse_ffn_layer(x, packed: PackedLayer, predictor: DevicePredictor, k: int,
                     dense_first_last: bool = True, has_comp: bool = True,
                     out: torch.Tensor | None = None, return_indices: bool = False,
                     workspace: torch.Tensor | None = None,
                     residual: torch.Tensor | None = None, x_next: torch.Tensor | None = None,
                     x_pred_f32: torch.Tensor | None = None,
                     logits_in: torch.Tensor | None = None, f32_out: bool = True,
                     mask_in: torch.Tensor | None = None):
    """One layer's FFN branch over every block of x (T, d); returns y (T, d) f32.

    Semantics of ``engine.py:254-310`` (mode "predicted"): blocks 0 and n-1 run
    dense when ``dense_first_last`` (``:258-262``; "first" / "last" for a sequence
    shard holding only the prompt's first / last block); k >= d_ffn runs every block
    dense with no predictor or compensator (``:268``); otherwise predictor ->
    top-k -> sparse FFN -> + compensator (``:284-300``).  Under tensor
    parallelism y is this rank's partial sum (all-reduce it, see ``tp.py``).
    With ``return_indices`` also returns the (n_predicted, k) global indices.
    ``residual`` (f32 (T, d), may be ``out``) fuses the residual add of
    ``engine.py:308`` into the down-projection epilogue; ``x_next`` (bf16 (T, d))
    receives bf16(y) as the next layer's input (tp_size == 1 only).
    ``x_pred_f32`` (f32 (T, d)) makes the predictor pool over f32 inputs (the
    reference's f32 RMSNorm output) instead of x; ``logits_in`` (f32 (T,)) are
    per-token predictor logits already produced by the FFN-input producer
    (``norm.rmsnorm(..., predictor=...)``), which skips the pooling's first pass.
    ``f32_out=False`` writes only the bf16 ``x_next`` (no f32 y; returned in its place):
    a tensor-parallel partial for a bf16 reduce-scatter.
    ``mask_in`` (int32 (n_blk, ceil(d_ffn / 32)) selection bitmasks, row b = block b, as
    ``predict_mask`` writes them) gives the selection instead of running the predictor:
    the sequence-parallel predictor under tensor parallelism (``tp.SeqParallelTP``), where
    each rank predicts its own blocks and the masks are all-gathered.
    """
    dev = packed.device
    if packed.d != packed.d_model:
        raise UnsupportedError(f"sparse_ffn_layer needs d_model % 64 == 0 (got {packed.d_model}); "
                               "the per-block drop-ins take any width")
    xb = _x_bf16(x, dev)
    T, d = xb.shape
    if d != packed.d or predictor.d != d or predictor.f != packed.f_global:
        raise ValidationError(f"layer shapes disagree: x {tuple(xb.shape)}, packed d={packed.d} "
                              f"f={packed.f_global}, predictor d={predictor.d} f={predictor.f}")
    if not 1 <= k <= packed.f_global:
        raise ValidationError(f"k={k} out of range [1, {packed.f_global}]")
    lib = _dev.lib_for(dev)
    if f32_out:
        y = out if out is not None else torch.empty((T, d), dtype=torch.float32, device=dev)
    else:
        if x_next is None or residual is not None:
            raise ValidationError("f32_out=False needs x_next (the bf16 output) and no residual")
        y = None
    n_blk = -(-T // BLOCK)
    dfl = dense_first_last_code(dense_first_last)
    if k >= packed.f_global:
        n_pred = 0
    else:
        n_pred = max(0, n_blk - (0 if dfl == 0 else 2 if dfl == 1 else 1))
    idx = None
    if return_indices and n_pred > 0:
        idx = torch.empty((n_pred, k), dtype=torch.int32, device=dev)
    ws_n = layer_workspace_bytes(T, packed, predictor.r, k, dense_first_last)
    ws = workspace if workspace is not None and workspace.numel() >= ws_n else \
        _dev.workspace(dev, ws_n)
    for name, t, shape, dt in (("x_pred_f32", x_pred_f32, (T, d), torch.float32),
                               ("logits_in", logits_in, (T,), torch.float32),
                               ("mask_in", mask_in, (n_blk, mask_words(packed.f_global)),
                                torch.int32)):
        if t is not None and (not t.is_cuda or t.dtype != dt or tuple(t.shape) != shape
                              or not t.is_contiguous()):
            raise ValidationError(f"{name} must be a contiguous CUDA {dt} tensor of shape {shape}")
    if mask_in is not None:
        if return_indices or x_pred_f32 is not None or logits_in is not None:
            raise ValidationError("mask_in replaces the predictor: no return_indices, "
                                  "x_pred_f32 or logits_in")
        _lib.check(lib.ffwd_ffn_layer_masked(
            xb.data_ptr(), T, d, packed.wgu_t.data_ptr(), packed.wd.data_ptr(), packed.f_local,
            packed.rc_local, packed.f_global, k, dfl, int(has_comp and packed.rc_local > 0),
            packed.tp_rank, packed.tp_size, mask_in.data_ptr(), mask_in.shape[1], _dev.ptr(y),
            _dev.ptr(residual), _dev.ptr(x_next), ws.data_ptr(), ws.numel(),
            _dev.stream_handle(dev)), "ffn_layer_masked")
        return y if y is not None else x_next
    _lib.check(lib.ffwd_ffn_layer2(
        xb.data_ptr(), T, d, packed.wgu_t.data_ptr(), packed.wd.data_ptr(), packed.f_local,
        packed.rc_local, predictor.query.data_ptr(), predictor.w1.data_ptr(),
        predictor.w2.data_ptr(), predictor.r, predictor.f, k, dfl,
        int(has_comp and packed.rc_local > 0), packed.tp_rank, packed.tp_size, _dev.ptr(y),
        _dev.ptr(residual), _dev.ptr(x_next), _dev.ptr(idx), k if idx is not None else 0,
        _dev.ptr(x_pred_f32), _dev.ptr(logits_in), ws.data_ptr(), ws.numel(),
        _dev.stream_handle(dev)), "ffn_layer")
    if y is None:
        y = x_next
    if return_indices:
        return y, idx
    return y


def mask_words(f: int) -> int:
    """32-bit words per selection bitmask row of d_ffn = f neurons."""
    return (f + 31) // 32


def predict_mask(x, predictor: DevicePredictor, k: int, blk_begin: int = 0,
                 blk_count: int | None = None, logits_in: torch.Tensor | None = None,
                 out: torch.Tensor | None = None,
                 workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Predictor + top-k of blocks [blk_begin, blk_begin + blk_count) of x (T, d) (bf16, or
    f32 for the reference's f32 predictor input), as selection bitmasks: int32
    (blk_count, ceil(d_ffn / 32)), bit j of word j // 32 = neuron j kept
    (``predictor.py:68-81`` -> ``build_mask``).  ``logits_in`` (f32 (T,)): the per-token
    logits from the FFN-input producer.  The indices are bit-identical to the ones
    ``sparse_ffn_layer`` selects for those blocks; the masks feed its ``mask_in``."""
    dev = predictor.w1.device
    xt = x if isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32 \
        else _x_bf16(x, dev)
    xt = xt.contiguous()
    T, d = xt.shape
    if d != predictor.d:
        raise ValidationError(f"x width {d} != predictor d_model {predictor.d}")
    n_blk = -(-T // BLOCK)
    if blk_count is None:
        blk_count = n_blk - blk_begin
    if not 1 <= k <= predictor.f:
        raise ValidationError(f"k={k} out of range [1, {predictor.f}]")
    w = mask_words(predictor.f)
    if out is None:
        out = torch.empty((blk_count, w), dtype=torch.int32, device=dev)
    if (not out.is_cuda or out.dtype != torch.int32 or out.dim() != 2 or out.shape[0] < blk_count
            or out.shape[1] != w or not out.is_contiguous()):
        raise ValidationError(f"out must be a contiguous CUDA int32 tensor of {blk_count} x {w}")
    if logits_in is not None and (not logits_in.is_cuda or logits_in.dtype != torch.float32
                                  or tuple(logits_in.shape) != (T,)):
        raise ValidationError(f"logits_in must be a CUDA float32 tensor of shape ({T},)")
    lib = _dev.lib_for(dev)
    ws_n = int(lib.ffwd_predict_mask_workspace_bytes(blk_count, d, predictor.r, predictor.f))
    ws = workspace if workspace is not None and workspace.numel() >= ws_n else \
        _dev.workspace(dev, ws_n)
    _lib.check(lib.ffwd_predict_mask(
        xt.data_ptr(), int(xt.dtype == torch.float32), T, d, blk_begin, blk_count,
        predictor.query.data_ptr(), predictor.w1.data_ptr(), predictor.w2.data_ptr(),
        predictor.r, predictor.f, k, _dev.ptr(logits_in), out.data_ptr(), w, ws.data_ptr(),
        ws.numel(), _dev.stream_handle(dev)), "predict_mask")
    return out


def mask_indices(mask: torch.Tensor, f: int) -> list:
    """Host helper: the ascending neuron ids of each bitmask row (int32 (n, ceil(f/32)))."""
    m = mask.cpu().numpy().view(np.uint32)
    bits = np.unpackbits(m.view(np.uint8), axis=1, bitorder="little")[:, :f]
    return [np.flatnonzero(row).astype(np.int64) for row in bits]


MODES = ("predicted", "oracle", "static")
_MODE_CODE = {"oracle": 1, "static": 2}


def oracle_scores(x, packed: PackedLayer) -> torch.Tensor:
    """Dense-scoring pass of ``oracle_experts`` over every 128-token block of x (T, d):
    H = silu(x Wg) * (x Wu) on the up-projection kernel, then per-block column norms
    (``hidden_column_scores``).  Returns f32 (n_blk, d_ffn).  tp_size 1 only."""
    if packed.tp_size != 1:
        raise ValidationError("oracle scoring needs the unsharded layer (tp_size 1)")
    dev = packed.device
    xb = _x_bf16(x, dev)
    T, d = xb.shape
    if d != packed.d_model:
        raise ValidationError(f"x width {d} != d_model {packed.d_model}")
    xb = _pad_cols(xb, packed.d)
    d = packed.d
    lib = _dev.lib_for(dev)
    f = packed.f_local
    n_blk = -(-T // BLOCK)
    out = torch.empty((n_blk, f), dtype=torch.float32, device=dev)
    ws = _dev.workspace(dev, lib.ffwd_hidden_scores_workspace_bytes(T, d, f))
    _lib.check(lib.ffwd_hidden_scores(xb.data_ptr(), T, d, packed.wgu_t.data_ptr(), f,
                                      packed.rc_local, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                      _dev.stream_handle(dev)), "hidden_scores")
    return out


def ffn_layer_mode(x, packed: PackedLayer, k: int, mode: str, dense_first_last: bool = True,
                   has_comp: bool = True, out: torch.Tensor | None = None,
                   residual: torch.Tensor | None = None, x_next: torch.Tensor | None = None,
                   return_indices: bool = False):
    """The FFN branch of ``engine.py:254-310`` in the ablation modes (tp_size 1).

    ``oracle``: each sparse block keeps the top-k of its own dense hidden norms
    (``oracle_experts``); ``static``: block 0 runs dense and its mask serves every later
    block (``FirstBlockStatic``, ``engine.py:272-283``).  Dense blocks and the full-K
    shortcut as in the engine.  Returns y (and the masks, int32 rows, with
    ``return_indices``: one row per sparse block for oracle, one row for static).
    """
    if mode not in _MODE_CODE:
        raise ValidationError(f"unknown mode {mode!r}; expected one of {tuple(_MODE_CODE)}")
    if packed.tp_size != 1:
        raise ValidationError("the ablation modes need the unsharded layer (tp_size 1)")
    if packed.d != packed.d_model:
        raise UnsupportedError(f"ffn_layer_mode needs d_model % 64 == 0 (got {packed.d_model})")
    dev = packed.device
    xb = _x_bf16(x, dev)
    T, d = xb.shape
    f = packed.f_local
    if not 1 <= k <= f:
        raise ValidationError(f"k={k} out of range [1, {f}]")
    lib = _dev.lib_for(dev)
    y = out if out is not None else torch.empty((T, d), dtype=torch.float32, device=dev)
    n_blk = -(-T // BLOCK)
    if mode == "static":
        n_rows = 1 if k < f else 0
    else:
        n_rows = 0 if k >= f else (max(0, n_blk - 2) if dense_first_last else n_blk)
    idx = torch.empty((max(n_rows, 1), k), dtype=torch.int32, device=dev) \
        if return_indices else None
    code = _MODE_CODE[mode]
    hc = int(has_comp and packed.rc_local > 0)
    ws = _dev.workspace(dev, lib.ffwd_ffn_layer_mode_workspace_bytes(
        T, d, f, packed.rc_local, k, code, int(dense_first_last)))
    _lib.check(lib.ffwd_ffn_layer_mode(
        xb.data_ptr(), T, d, packed.wgu_t.data_ptr(), packed.wd.data_ptr(), f, packed.rc_local,
        k, code, int(dense_first_last), hc, y.data_ptr(), _dev.ptr(residual), _dev.ptr(x_next),
        _dev.ptr(idx), k if idx is not None else 0, ws.data_ptr(), ws.numel(),
        _dev.stream_handle(dev)), "ffn_layer_mode")
    if return_indices:
        return y, idx[:n_rows]
    return y


def set_raster(up_group: int, down_group: int) -> None:
    """Blocks per L2 raster group of the up / down gather-GEMMs (tuning knob)."""
    _lib.check(_lib.load_library().ffwd_set_raster(up_group, down_group), "set_raster")


STAGES = ("pool", "predictor_w1", "predictor_w2", "topk", "plan", "up_proj", "down_proj",
          "ffn_norm")


def timing_enable(on: bool = True) -> None:
    """Record CUDA events around every kernel launch of ``sparse_ffn_layer``."""
    _lib.load_library().ffwd_timing_enable(int(on))


def timing_read() -> dict:
    """{stage: (summed ms, launches)} since the last read (waits for the events)."""
    import ctypes
    n = len(STAGES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int * n)()
    _lib.check(_lib.load_library().ffwd_timing_read(ms, cnt, n), "timing_read")
    return {STAGES[i]: (ms[i], cnt[i]) for i in range(n)}
