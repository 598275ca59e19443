"""Tensor parallelism over d_ffn.

Rank s of N holds the neurons {j : j % N == s} (strided, so planted
contiguous neuron groups spread evenly) of W_gate / W_up / W_down and a
contiguous 1/N slice of the compensator bottleneck.  The predictor is
replicated: every rank computes the same global top-k (bit-exact, so no
collective is needed before the FFN) and keeps its local subset.  Each rank's
down projection yields a partial Y; one all-reduce (sum) per layer completes
it -- either NCCL (``allreduce_partial``) or the fused peer-memory kernel
(``PeerBuffers.complete``: reduce-scatter + all-gather over NVLink in one pass,
with the residual add and the next layer's bf16 input fused in), or that same
completion overlapped with the down projection block by block
(``PeerBuffers.layer_overlap``: K3 publishes per-block tile counts, the completion
drains each block as soon as every rank has finished it).  Independent
prompts are data parallel and need no collective at all.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _dev, _lib
from .compensator import CompensatorParams
from .errors import ValidationError
from .layer import (BLOCK, PackedLayer, dense_first_last_code, layer_workspace_bytes,
                    mask_words, pack_layer, predict_mask, shard_comp_cols, shard_neurons,
                    sparse_ffn_layer)
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


# ---------------------------------------------------------------- fused completion
def allreduce_residual_fused(partials, outs, flags, rank: int, residual: torch.Tensor,
                             epoch: int, xnexts=None, max_ctas: int = 0) -> None:
    """One rank's fused TP completion (``ffwd_allreduce_residual``): for its row slice,
    out_p = residual + sum_q partial_q on every rank p, over peer pointers.

    ``partials`` / ``outs`` / ``flags`` / ``xnexts``: one entry per rank, each a CUDA
    tensor (single-process emulation) or an int device pointer (peer mappings from
    ``PeerBuffers``).  ``epoch`` increases by one per call.
    """
    import ctypes
    from . import _dev, _lib
    n = len(partials)
    if not (len(outs) == len(flags) == n) or (xnexts is not None and len(xnexts) != n):
        raise ValidationError("one partial, out, flag (and x_next) buffer per rank")
    T, d = residual.shape

    def ptrs(items):
        arr = (ctypes.c_void_p * n)()
        for i, t in enumerate(items):
            arr[i] = t if isinstance(t, int) else t.data_ptr()
        return arr

    lib = _dev.lib_for(residual.device)
    _lib.check(lib.ffwd_allreduce_residual(
        ptrs(partials), ptrs(outs), ptrs(xnexts) if xnexts is not None else None, ptrs(flags),
        n, rank, residual.data_ptr(), T, d, int(epoch) & 0xFFFFFFFF, max_ctas,
        _dev.stream_handle(residual.device)), "allreduce_residual")


def _ptr_array(items):
    import ctypes
    arr = (ctypes.c_void_p * len(items))()
    for i, t in enumerate(items):
        arr[i] = t if isinstance(t, int) else t.data_ptr()
    return arr


def sparse_ffn_layer_tp_overlap(x, packed: PackedLayer, predictor: DevicePredictor, k: int, *,
                                partials, outs, flags, y_done, residual: torch.Tensor,
                                epoch: int, y_epoch: int, xnexts=None,
                                dense_first_last: bool = True, has_comp: bool = True,
                                comm_ctas: int = 32, x_pred_f32=None, logits_in=None,
                                workspace: torch.Tensor | None = None, comm_stream=None):
    """One rank's TP layer with the completion overlapped (``ffwd_ffn_layer_tp_overlap``).

    The down projection writes this rank's partial Y into ``partials[rank]`` and counts
    finished column tiles per block in ``y_done[rank]``; a completion kernel on
    ``comm_stream`` sums each block over the ranks (fixed rank order, + ``residual``)
    into every rank's ``outs`` (and ``xnexts``) while later blocks are still computed.
    Peer lists hold one CUDA tensor (single-process emulation) or device pointer
    (``PeerBuffers``) per rank.  The current stream waits for the completion.
    """
    from .layer import _x_bf16
    dev = packed.device
    xb = _x_bf16(x, dev)
    T, d = xb.shape
    n = packed.tp_size
    if not (len(partials) == len(outs) == len(flags) == len(y_done) == n) or (
            xnexts is not None and len(xnexts) != n):
        raise ValidationError("one partial, out, flag, y_done (and x_next) buffer per rank")
    if tuple(residual.shape) != (T, d) or residual.dtype != torch.float32:
        raise ValidationError(f"residual must be f32 {(T, d)}")
    ws_n = layer_workspace_bytes(T, packed, predictor.r, k, dense_first_last)
    ws = workspace if workspace is not None and workspace.numel() >= ws_n else \
        _dev.workspace(dev, ws_n)
    cs = comm_stream if comm_stream is not None else torch.cuda.Stream(dev)
    lib = _dev.lib_for(dev)
    _lib.check(lib.ffwd_ffn_layer_tp_overlap(
        xb.data_ptr(), T, d, packed.wgu_t.data_ptr(), packed.wd.data_ptr(), packed.f_local,
        packed.rc_local, predictor.query.data_ptr(), predictor.w1.data_ptr(),
        predictor.w2.data_ptr(), predictor.r, predictor.f, k,
        dense_first_last_code(dense_first_last),
        int(has_comp and packed.rc_local > 0), packed.tp_rank, n, None, 0,
        _dev.ptr(x_pred_f32), _dev.ptr(logits_in), _ptr_array(partials), _ptr_array(outs),
        _ptr_array(xnexts) if xnexts is not None else None, _ptr_array(flags),
        _ptr_array(y_done), residual.data_ptr(), int(epoch) & 0xFFFFFFFF,
        int(y_epoch) & 0xFFFFFFFF, comm_ctas, ws.data_ptr(), ws.numel(),
        _dev.stream_handle(dev), cs.cuda_stream), "ffn_layer_tp_overlap")


class PeerBuffers:
    """Per-rank partial-Y, residual-stream and flag buffers shared over CUDA IPC, for the
    fused TP completion (one process per GPU, NVLink peer access)."""

    def __init__(self, T: int, d: int, device, group=None, with_xnext: bool = True):
        import ctypes
        from . import _lib
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        dev = torch.device(device)
        self.partial = torch.empty((T, d), dtype=torch.float32, device=dev)
        self.out = torch.empty((T, d), dtype=torch.float32, device=dev)
        self.xnext = torch.empty((T, d), dtype=torch.bfloat16, device=dev) if with_xnext else None
        self.flags = torch.zeros((2 * self.world + 1,), dtype=torch.int32, device=dev)
        # per-block finished down tiles (overlapped completion); never reset
        self.y_done = torch.zeros((-(-T // BLOCK),), dtype=torch.int32, device=dev)
        lib = _lib.load_library()
        mine = []
        for t in (self.partial, self.out, self.xnext, self.flags, self.y_done):
            if t is None:
                mine.append(None)
                continue
            h = (ctypes.c_char * 64)()
            off = ctypes.c_size_t()
            _lib.check(lib.ffwd_ipc_get_handle(t.data_ptr(), h, ctypes.byref(off)), "ipc handle")
            mine.append((bytes(h), off.value))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        self.peer = {"partial": [], "out": [], "xnext": [], "flags": [], "y_done": []}
        bases: dict = {}  # one mapping per peer allocation (tensors may share a segment)
        for p in range(self.world):
            for key, t, hv in zip(("partial", "out", "xnext", "flags", "y_done"),
                                  (self.partial, self.out, self.xnext, self.flags, self.y_done),
                                  allh[p]):
                if hv is None:
                    continue
                if p == self.rank:
                    self.peer[key].append(t.data_ptr())
                    continue
                if (p, hv[0]) not in bases:
                    base = ctypes.c_void_p()
                    _lib.check(lib.ffwd_ipc_open(hv[0], ctypes.byref(base)), "ipc open")
                    self._opened.append(base.value)
                    bases[(p, hv[0])] = base.value
                self.peer[key].append(bases[(p, hv[0])] + hv[1])
        self.epoch = 0
        self.y_epoch = 0
        self.comm_stream = torch.cuda.Stream(dev)
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)

    def complete(self, residual: torch.Tensor, max_ctas: int = 0) -> torch.Tensor:
        """After this rank's down projection wrote ``self.partial``: every rank's ``out``
        becomes residual + sum of partials (and ``xnext`` its bf16 copy)."""
        self.epoch += 1
        allreduce_residual_fused(self.peer["partial"], self.peer["out"], self.peer["flags"],
                                 self.rank, residual, self.epoch,
                                 self.peer["xnext"] if self.xnext is not None else None,
                                 max_ctas)
        return self.out

    def layer_overlap(self, x, packed: PackedLayer, predictor: DevicePredictor, k: int,
                      residual: torch.Tensor, dense_first_last: bool = True,
                      comm_ctas: int = 32, **kw) -> torch.Tensor:
        """This rank's layer with the completion overlapped with its down projection:
        afterwards every rank's ``out`` holds residual + the full FFN output (``xnext``
        its bf16 copy; it must not be the layer input ``x``)."""
        self.epoch += 1
        self.y_epoch += 1
        sparse_ffn_layer_tp_overlap(
            x, packed, predictor, k, partials=self.peer["partial"], outs=self.peer["out"],
            flags=self.peer["flags"], y_done=self.peer["y_done"], residual=residual,
            epoch=self.epoch, y_epoch=self.y_epoch,
            xnexts=self.peer["xnext"] if self.xnext is not None else None,
            dense_first_last=dense_first_last, comm_ctas=comm_ctas,
            comm_stream=self.comm_stream, **kw)
        return self.out

    def close(self):
        from . import _lib
        lib = _lib.load_library()
        for p in self._opened:
            lib.ffwd_ipc_close(p)
        self._opened = []


# ------------------------------------------------- sequence-parallel residual (RS / AG)
class TorchComm:
    """The two collectives of the sequence-parallel TP layer over ``torch.distributed``
    (NCCL over NVLink on the GPU box; gloo for CPU tests)."""

    def __init__(self, group=None):
        self.group = group
        # gloo has no CUDA all-gather / reduce-scatter: stage through host memory (the
        # single-GPU functional emulation of the bench; NCCL takes device tensors)
        self.staged = dist.get_backend(group) == "gloo"

    def _run(self, fn, out, inp):
        if self.staged and out.is_cuda:
            o, i = out.cpu(), inp.cpu()
            if o.dtype == torch.bfloat16:  # gloo reductions of bf16: widen on the host
                o, i = o.float(), i.float()
            fn(o, i, group=self.group)
            out.copy_(o)
        else:
            fn(out, inp, group=self.group)

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        self._run(dist.all_gather_into_tensor, out, inp)

    def all_gather_start(self, out: torch.Tensor, inp: torch.Tensor):
        """Start an all-gather that overlaps the caller's next kernels (NCCL runs it on its
        own stream); returns a handle whose ``wait()`` orders the current stream after it.
        Host-staged (gloo) gathers complete before returning."""
        if self.staged and out.is_cuda:
            self.all_gather(out, inp)
            return None
        return dist.all_gather_into_tensor(out, inp, group=self.group, async_op=True)

    def reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        self._run(lambda o, i, group: dist.reduce_scatter_tensor(o, i, op=dist.ReduceOp.SUM,
                                                                 group=group), out, inp)


def seq_rows(T: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) of the residual stream rank `rank` owns (T % world == 0)."""
    if T % world:
        raise ValidationError(f"{T} tokens do not split evenly over {world} ranks")
    n = T // world
    return rank * n, (rank + 1) * n


class SeqParallelTP:
    """Tensor parallelism over d_ffn with a sequence-parallel residual stream.

    The FFN branch of ``engine.py:263-308`` split over N ranks.  Rank r owns rows
    [r T/N, (r+1) T/N) of the f32 residual stream h and the strided d_ffn shard
    {j : j % N == r} of every layer (``pack_layer(..., tp_rank=r, tp_size=N)``).  Per layer:

      1. ``norm``: h[R_r] += y[R_r] (the previous layer's reduced FFN output,
         ``engine.py:308``) and x[R_r] = rmsnorm(h[R_r]) with the predictor's per-token
         logits -- one kernel (``ffwd_rmsnorm_ex`` with ``add``) on T/N rows;
      2. ``predict`` (sequence-parallel predictor, when T/N is a whole number of 128-token
         blocks): the predictor and top-k of this rank's own blocks only
         (``predictor.py:68-81`` is block-local), written as selection bitmasks
         (``layer.predict_mask``: ceil(d_ffn / 32) words per block);
      3. ``gather``: all-gather x (bf16 [T x d]; started before ``predict`` so the transfer
         overlaps the rank's predictor) and the bitmasks ([n_blk x words]), or, with a
         replicated predictor, x and the f32 logits;
      4. ``ffn``: the FFN branch over all T tokens on this rank's shard: each rank keeps its
         own neurons of every block's selection (``mask_in``; replicated predictor: every
         rank recomputes the same global top-k, bit-exact) -> partial y (f32, or bf16 with
         ``reduce_dtype=torch.bfloat16``);
      5. ``scatter``: reduce-scatter the partial y -> y[R_r].

    ``finish`` adds the last layer's y.  NVLink bytes per rank and layer:
    (N-1)/N T d (2 + 4) (bf16 all-gather + f32 reduce-scatter; 2 + 2 with a bf16 reduce)
    plus n_blk d_ffn / 8 bytes of bitmasks, against (N-1)/N T d 8 for an f32 all-reduce;
    the norm, the logits and the predictor run on T/N rows instead of T.

    The phases are separate methods so a single process can drive N emulated ranks in
    lockstep (tests); ``layer`` runs them with the real collectives.  ``norm_fn`` /
    ``predict_fn`` / ``ffn_fn`` replace the GPU kernels (CPU tests: the oracle);
    ``ffn_fn(l, x_full, sel_full, y_part)`` gets the gathered bitmasks (sharded predictor)
    or logits (replicated)."""

    def __init__(self, layers, T: int, d: int, rank: int, world: int, device,
                 comm=None, gain=None, reduce_dtype=torch.float32, dense_first_last=True,
                 norm_fn=None, ffn_fn=None, x_dtype=torch.bfloat16, predict_fn=None,
                 shard_predictor=None, f: int | None = None):
        if reduce_dtype not in (torch.float32, torch.bfloat16):
            raise ValidationError("reduce_dtype must be float32 or bfloat16")
        self.layers = layers  # [(packed shard, DevicePredictor, k)] (CPU tests: (None, None, k))
        self.T, self.d, self.rank, self.world = T, d, rank, world
        self.r0, self.r1 = seq_rows(T, rank, world)
        dev = torch.device(device)
        self.dev = dev
        if comm is None and dist.is_available() and dist.is_initialized():
            comm = TorchComm()
        self.comm = comm  # None: a lockstep driver moves the data between the phases
        self.reduce_dtype = reduce_dtype
        self.dense_first_last = dense_first_last
        n = self.r1 - self.r0
        self.gain = gain if gain is not None else torch.ones(d, device=dev)
        self.x_shard = torch.empty((n, d), dtype=x_dtype, device=dev)
        self.lg_shard = torch.empty((n,), dtype=torch.float32, device=dev)
        self.x_full = torch.empty((T, d), dtype=x_dtype, device=dev)
        self.lg_full = torch.empty((T,), dtype=torch.float32, device=dev)
        self.y_part = torch.empty((T, d), dtype=reduce_dtype, device=dev)
        self.y_shard = torch.empty((n, d), dtype=reduce_dtype, device=dev)
        # sequence-parallel predictor: this rank's rows must be whole blocks.  Default: on
        # from 4 ranks, where the replicated predictor's share of a rank's layer is
        # largest (single-GPU proxy, tools/tp_rank_proxy.py: -4% at TP=4, -8% at TP=8)
        whole = T % (BLOCK * world) == 0
        if shard_predictor and not whole:
            raise ValidationError(f"a sharded predictor needs T % (128 x {world}) == 0, T={T}")
        self.shard_predictor = (whole and world >= 4) if shard_predictor is None \
            else bool(shard_predictor)
        self.n_blk = -(-T // BLOCK)
        if f is None:
            f = next((lay[1].f for lay in layers if lay is not None and lay[1] is not None), None)
        if self.shard_predictor:
            if f is None:
                raise ValidationError("the sharded predictor needs d_ffn (f)")
            w = mask_words(f)
            self.mask_shard = torch.zeros((self.n_blk // world, w), dtype=torch.int32, device=dev)
            self.mask_full = torch.zeros((self.n_blk, w), dtype=torch.int32, device=dev)
        self.f = f
        self.norm_fn = norm_fn or self._gpu_norm
        self.predict_fn = predict_fn or self._gpu_predict
        self.ffn_fn = ffn_fn or self._gpu_ffn
        self.workspace = None
        self.pending = False  # y_shard holds a layer output not yet added to h

    # -- which of this rank's blocks run the predictor (engine.py:258-262, :268)
    def predicted_blocks(self, k: int) -> tuple[int, int]:
        """Shard-relative block range [lo, hi) of this rank's predicted blocks."""
        nbr = self.n_blk // self.world
        if self.f is not None and k >= self.f:
            return 0, 0  # full-K shortcut: every block dense
        g0, g1 = self.rank * nbr, (self.rank + 1) * nbr
        if dense_first_last_code(self.dense_first_last):
            g0, g1 = max(g0, 1), min(g1, self.n_blk - 1)
        return (g0 - self.rank * nbr, g1 - self.rank * nbr) if g1 > g0 else (0, 0)

    # -- default (GPU) compute
    def _gpu_norm(self, l, h_shard, add):
        from .norm import rmsnorm
        rmsnorm(h_shard, self.gain, out=self.x_shard, predictor=self.layers[l][1],
                logits=self.lg_shard, add=add)

    def _gpu_predict(self, l, lo, hi):
        _, dp, k = self.layers[l]
        predict_mask(self.x_shard, dp, k, blk_begin=lo, blk_count=hi - lo,
                     logits_in=self.lg_shard, out=self.mask_shard[lo:hi])

    def _gpu_ffn(self, l, x_full, sel_full, y_part):
        packed, dp, k = self.layers[l]
        if self.workspace is None:
            n = max(layer_workspace_bytes(self.T, p, q.r, kk, self.dense_first_last)
                    for p, q, kk in self.layers)
            self.workspace = torch.empty(n, dtype=torch.uint8, device=self.dev)
        sel = ({"mask_in": sel_full} if self.shard_predictor else {"logits_in": sel_full})
        if y_part.dtype == torch.float32:
            sparse_ffn_layer(x_full, packed, dp, k, out=y_part, workspace=self.workspace,
                             dense_first_last=self.dense_first_last, **sel)
        else:
            sparse_ffn_layer(x_full, packed, dp, k, x_next=y_part, f32_out=False,
                             workspace=self.workspace, dense_first_last=self.dense_first_last,
                             **sel)

    # -- phases
    def norm(self, l: int, h_shard: torch.Tensor) -> None:
        self.norm_fn(l, h_shard, self.y_shard if self.pending else None)
        self.pending = False

    def predict(self, l: int) -> None:
        if not self.shard_predictor:
            return
        lo, hi = self.predicted_blocks(self.layers[l][2])
        if hi > lo:
            self.predict_fn(l, lo, hi)

    def gather(self) -> None:
        self.comm.all_gather(self.x_full, self.x_shard)
        self.gather_selection()

    def gather_selection(self) -> None:
        if self.shard_predictor:
            self.comm.all_gather(self.mask_full, self.mask_shard)
        else:
            self.comm.all_gather(self.lg_full, self.lg_shard)

    def ffn(self, l: int) -> None:
        self.ffn_fn(l, self.x_full, self.mask_full if self.shard_predictor else self.lg_full,
                    self.y_part)

    def scatter(self) -> None:
        self.comm.reduce_scatter(self.y_shard, self.y_part)
        self.pending = True

    def finish(self, h_shard: torch.Tensor) -> torch.Tensor:
        if self.pending:
            h_shard.add_(self.y_shard.to(h_shard.dtype))
            self.pending = False
        return h_shard

    def layer(self, l: int, h_shard: torch.Tensor) -> None:
        self.norm(l, h_shard)
        # the all-gather of the FFN input (T d bf16, the layer's largest transfer before the
        # FFN) overlaps this rank's predictor; the small selection gather follows it
        start = getattr(self.comm, "all_gather_start", None)
        work = start(self.x_full, self.x_shard) if start else None
        if start is None:
            self.comm.all_gather(self.x_full, self.x_shard)
        self.predict(l)
        self.gather_selection()
        if work is not None:
            work.wait()
        self.ffn(l)
        self.scatter()

    def stack(self, h_shard: torch.Tensor) -> torch.Tensor:
        """Every layer over this rank's residual rows (h_shard f32 [T/N x d], in place)."""
        for l in range(len(self.layers)):
            self.layer(l, h_shard)
        return self.finish(h_shard)
