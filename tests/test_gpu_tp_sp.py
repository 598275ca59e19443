"""Tensor parallelism with the sequence-parallel residual (tp.SeqParallelTP), emulated on
one GPU: N = 2 / 4 / 8 ranks driven in lockstep in one process, each with its own strided
d_ffn shard, its own T/N residual rows and its own buffers; the all-gather and the
reduce-scatter are done by the test (concatenation; a sum in rank order).  The real run
(bench.py --gpus N) does the same phases with NCCL between them.

Checks against the unsharded stack (N = 1, the bench's single-GPU path):
  * the gathered FFN input and predictor logits of the first layer are bit-identical
    (the RMSNorm and its fused logits are row-local);
  * every rank's replicated predictor selects the unsharded layer's indices, bit for bit;
  * the first layer's output equals the unsharded one up to f32 reassociation of the
    N partial sums (rel-L2 <= 1e-5; bf16 reduce: the parity tolerance 5e-3), and with the
    f32 reduce the two-layer stack stays within the parity tolerance (a bf16 reduce
    rounds every layer's output, which moves the next layer's input and can flip its
    boundary neurons: the one-layer bound is its parity statement).
"""

import numpy as np
import pytest
import torch

from oracle import ffwd_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ff():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_00397_b200 as ff
    from paper_2602_00397_b200 import _lib
    _lib.require_device(torch.cuda.current_device())
    return ff


D, F, T, L = 2048, 8192, 4096, 2


def host_model():
    out = []
    for l in range(L):
        rng = np.random.default_rng([404, l])
        w = {n: orc.bf16_round(rng.standard_normal(s, dtype=np.float32) * np.float32(0.02))
             for n, s in (("w_gate", (D, F)), ("w_up", (D, F)), ("w_down", (F, D)))}
        pred = orc.init_predictor(np.random.default_rng([404, l, 1]), D, F)
        comp = {k: orc.bf16_round(v) for k, v in
                orc.init_compensator(np.random.default_rng([404, l, 2]), D).items()}
        out.append((w, pred, comp, orc.budget_to_k(0.5, F)))
    return out


def run_emulated(ff, model, world, reduce_dtype, n_layers=L, shard_predictor=False):
    from paper_2602_00397_b200.tp import SeqParallelTP, seq_rows
    dps = [ff.DevicePredictor.from_params(ff.PredictorParams(**p), "cuda") for _, p, _, _ in model]
    sps = []
    for r in range(world):
        layers = [(ff.pack_layer(w["w_gate"], w["w_up"], w["w_down"],
                                 ff.CompensatorParams(**c), device="cuda", tp_rank=r,
                                 tp_size=world), dps[l], k)
                  for l, (w, _, c, k) in enumerate(model[:n_layers])]
        sps.append(SeqParallelTP(layers, T, D, r, world, "cuda", comm=None,
                                 reduce_dtype=reduce_dtype, shard_predictor=shard_predictor))
    x0 = torch.randn((T, D), generator=torch.Generator().manual_seed(9)).to(
        torch.bfloat16).float().cuda()
    h = [x0[slice(*seq_rows(T, r, world))].clone() for r in range(world)]
    first = {}
    for l in range(n_layers):
        for r in range(world):
            sps[r].norm(l, h[r])
            sps[r].predict(l)                             # own blocks only (sharded)
        x_full = torch.cat([sp.x_shard for sp in sps])   # all-gather
        lg_full = torch.cat([sp.lg_shard for sp in sps])
        if shard_predictor:
            mask_full = torch.cat([sp.mask_shard for sp in sps])
        for sp in sps:
            sp.x_full.copy_(x_full)
            sp.lg_full.copy_(lg_full)
            if shard_predictor:
                sp.mask_full.copy_(mask_full)
            sp.ffn(l)
        total = sps[0].y_part.float().clone()            # reduce-scatter, rank order
        for sp in sps[1:]:
            total += sp.y_part.float()
        for r, sp in enumerate(sps):
            sp.y_shard.copy_(total[slice(*seq_rows(T, r, world))])
            sp.pending = True
        if l == 0:
            idx = []
            for sp in sps:  # each rank's global selection from the gathered input
                packed, dp, k = sp.layers[0]
                _, ir = ff.sparse_ffn_layer(x_full, packed, dp, k, logits_in=lg_full,
                                            return_indices=True)
                idx.append(ir)
            first = {"x": x_full.clone(), "lg": lg_full.clone(), "idx": idx,
                     "mask": mask_full.clone() if shard_predictor else None}
    for r, sp in enumerate(sps):
        sp.finish(h[r])
    torch.cuda.synchronize()
    return torch.cat(h), first


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("reduce", ["f32", "bf16"])
def test_seq_parallel_tp_matches_unsharded(ff, world, reduce):
    model = host_model()
    rd = torch.float32 if reduce == "f32" else torch.bfloat16
    h1, ref = run_emulated(ff, model, 1, torch.float32)
    hn, got = run_emulated(ff, model, world, rd)
    assert torch.equal(got["x"], ref["x"]), "gathered FFN input differs"
    assert torch.equal(got["lg"], ref["lg"]), "gathered predictor logits differ"
    for r, ir in enumerate(got["idx"]):
        assert torch.equal(ir, ref["idx"][0]), f"rank {r} selected different neurons"
    # one layer: f32 reassociation of the partials only
    h1a, _ = run_emulated(ff, model, 1, torch.float32, n_layers=1)
    hna, _ = run_emulated(ff, model, world, rd, n_layers=1)
    x0 = torch.randn((T, D), generator=torch.Generator().manual_seed(9)).to(
        torch.bfloat16).float().cuda()
    y1, yn = (h1a - x0).double(), (hna - x0).double()
    rel1 = float((yn - y1).norm() / y1.norm())
    assert rel1 <= (1e-5 if reduce == "f32" else 5e-3), rel1
    if reduce == "f32":  # the bf16 reduce's per-layer rounding moves later layers' inputs
        rel = float((hn - h1).double().norm() / h1.double().norm())
        assert rel <= 5e-3, rel


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_predictor_matches_replicated(ff, world):
    """The sequence-parallel predictor (each rank predicts only its own T/N rows' blocks,
    the selection bitmasks are all-gathered) gives every block the unsharded layer's
    indices bit for bit, and the stack the same output as the replicated predictor."""
    model = host_model()
    h_rep, rep = run_emulated(ff, model, world, torch.float32)
    h_sh, sh = run_emulated(ff, model, world, torch.float32, shard_predictor=True)
    n_pred = T // 128 - 2
    rows = ff.mask_indices(sh["mask"][1:1 + n_pred], F)  # blocks 1 .. n-2 are predicted
    want = rep["idx"][0].cpu().numpy()
    assert len(rows) == want.shape[0]
    for b, row in enumerate(rows):
        assert np.array_equal(row, want[b]), f"block {b + 1}: gathered mask != selection"
    assert torch.equal(h_sh, h_rep), "sharded and replicated predictors differ"


def test_predict_mask_and_mask_in_reproduce_the_layer(ff):
    """One GPU: ``predict_mask`` over a block range equals the indices the layer selects
    for those blocks, and ``sparse_ffn_layer(mask_in=...)`` (the selection given) is
    bit-identical to the layer running its own predictor (tp_size 1 and a TP=2 shard)."""
    w, pred, comp, k = host_model()[0]
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    x = torch.randn((T, D), generator=torch.Generator().manual_seed(3)).to(torch.bfloat16).cuda()
    n_blk = T // 128
    mask = torch.zeros((n_blk, ff.mask_words(F)), dtype=torch.int32, device="cuda")
    ff.predict_mask(x, dp, k, blk_begin=1, blk_count=5, out=mask[1:6])
    ff.predict_mask(x, dp, k, blk_begin=6, blk_count=n_blk - 7, out=mask[6:n_blk - 1])
    for tp_size in (1, 2):
        for rank in range(tp_size):
            packed = ff.pack_layer(w["w_gate"], w["w_up"], w["w_down"], ff.CompensatorParams(**comp),
                                   device="cuda", tp_rank=rank, tp_size=tp_size)
            y_ref, idx = ff.sparse_ffn_layer(x, packed, dp, k, return_indices=True)
            y_m = ff.sparse_ffn_layer(x, packed, dp, k, mask_in=mask)
            assert torch.equal(y_m, y_ref), (tp_size, rank)
    rows = ff.mask_indices(mask[1:n_blk - 1], F)
    for b, row in enumerate(rows):
        assert np.array_equal(row, idx[b].cpu().numpy()), b
    with pytest.raises(ff.errors.ValidationError):
        ff.sparse_ffn_layer(x, packed, dp, k, mask_in=mask[:, :3].contiguous())
