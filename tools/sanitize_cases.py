"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): every hot-path
kernel at parity sizes, checked against the oracle so a silent corruption also fails.

  cfg1   one predicted layer (d512 f1376 T1024): logits/pool, W1 cluster split-K (DSMEM), W2,
         top-k, plan, K2 (CTA pairs, multicast), K3 (per-block K2->K3 counters, PDL)
  edge   short / single-token blocks, k = 1, k = f - 1, ragged compensator, 64-col tiles
  norm   the FFN-input RMSNorm with fused logits and residual add
  mask   the sequence-parallel predictor's halves: predict_mask over a block range (top-k
         with bitmask output) and the masked layer at TP=2 (bitmask-to-list kernel)
  tp1    the fused TP completion kernel with one rank (the sanitizer serialises kernel
         launches, so two emulated ranks that wait on each other cannot both run under it;
         the two-rank flag protocol is covered by tests/test_gpu_tp_fused.py)
usage: python tools/sanitize_cases.py [case ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_00397_b200 as ff  # noqa: E402
from oracle import ffwd_oracle as orc  # noqa: E402


def layer(d, f, T, k, dfl, seed):
    rng = np.random.default_rng(seed)
    lw = orc.random_layer(rng, d, f, 0.02)
    for key in ("w_gate", "w_up", "w_down"):
        lw[key] = orc.bf16_round(lw[key])
    pred = orc.init_predictor(np.random.default_rng([seed, 1]), d, f)
    comp = {n: orc.bf16_round(v) for n, v in
            orc.init_compensator(np.random.default_rng([seed, 2]), d).items()}
    x = orc.bf16_round(rng.standard_normal((T, d)).astype(np.float32))
    packed = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], ff.CompensatorParams(**comp),
                           device="cuda")
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    y, idx = ff.sparse_ffn_layer(torch.from_numpy(x).to("cuda", torch.bfloat16), packed, dp, k,
                                 dense_first_last=dfl, return_indices=True)
    torch.cuda.synchronize()
    want, masks, _ = orc.ffn_layer_blockwise(x, lw, pred, comp, k, dfl, keep_masks=True)
    if masks:
        got = idx.cpu().numpy()
        for row, j in enumerate(sorted(masks)):
            assert np.array_equal(got[row], masks[j]), f"block {j} indices"
    y = y.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(y - want) / np.linalg.norm(want)
    assert rel < 5e-3, rel
    print(f"layer d{d} f{f} T{T} k{k}: ok (rel-L2 {rel:.2e})")


def case_cfg1():
    layer(512, 1376, 1024, 688, True, 2026)


def case_edge():
    for d, f, T, k, dfl in ((192, 520, 129, 259, True), (192, 520, 300, 1, False),
                            (192, 520, 300, 519, False), (320, 1000, 400, 333, True)):
        layer(d, f, T, k, dfl, d * 7 + T)


def case_norm():
    from paper_2602_00397_b200.norm import rmsnorm
    T, d = 300, 4096
    x = torch.randn((T, d), device="cuda")
    add = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    pred = orc.init_predictor(np.random.default_rng(3), d, 1024)
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    xb, x32, lg = rmsnorm(x, torch.ones(d, device="cuda"), out_f32=True, predictor=dp, add=add)
    torch.cuda.synchronize()
    from paper_2602_00397_b200.predictor import predictor_logits
    assert torch.equal(lg, predictor_logits(dp, xb))
    # ~10 rows per CTA: the row ring and the reduction slots wrap several times
    x2 = torch.randn((3000, d), device="cuda")
    xb2, _, lg2 = rmsnorm(x2, torch.ones(d, device="cuda"), predictor=dp)
    torch.cuda.synchronize()
    assert torch.equal(lg2, predictor_logits(dp, xb2))
    print("norm: ok")


def case_mask():
    d, f, T = 512, 1376, 1024
    k = ff.budget_to_k(0.5, f)
    rng = np.random.default_rng(77)
    lw = orc.random_layer(rng, d, f, 0.02)
    for key in ("w_gate", "w_up", "w_down"):
        lw[key] = orc.bf16_round(lw[key])
    pred = orc.init_predictor(np.random.default_rng([77, 1]), d, f)
    comp = {n: orc.bf16_round(v) for n, v in
            orc.init_compensator(np.random.default_rng([77, 2]), d).items()}
    x = torch.from_numpy(orc.bf16_round(rng.standard_normal((T, d)).astype(np.float32)))
    x = x.to("cuda", torch.bfloat16)
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    n_blk = T // 128
    mask = torch.zeros((n_blk, ff.mask_words(f)), dtype=torch.int32, device="cuda")
    ff.predict_mask(x, dp, k, blk_begin=1, blk_count=n_blk - 2, out=mask[1:n_blk - 1])
    for rank in range(2):
        packed = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], ff.CompensatorParams(**comp),
                               device="cuda", tp_rank=rank, tp_size=2)
        y_ref = ff.sparse_ffn_layer(x, packed, dp, k)
        y_m = ff.sparse_ffn_layer(x, packed, dp, k, mask_in=mask)
        torch.cuda.synchronize()
        assert torch.equal(y_m, y_ref), rank
    print("mask (predict_mask + masked TP=2 layer): ok")


def case_tp1():
    from paper_2602_00397_b200.tp import allreduce_residual_fused
    n, T, d = 1, 300, 256
    partials = [torch.randn((T, d), device="cuda") for _ in range(n)]
    residual = torch.randn((T, d), device="cuda")
    want = residual + partials[0]
    flags = [torch.zeros(2 * n + 1, dtype=torch.int32, device="cuda") for _ in range(n)]
    outs = [residual.clone() for _ in range(n)]
    streams = [torch.cuda.Stream() for _ in range(n)]
    for r in range(n):
        with torch.cuda.stream(streams[r]):
            allreduce_residual_fused(partials, outs, flags, r, outs[r], 1, None, max_ctas=16)
    torch.cuda.synchronize()
    assert all(torch.equal(o, want) for o in outs)
    print("tp1 fused completion: ok")


if __name__ == "__main__":
    cases = sys.argv[1:] or ["cfg1", "edge", "norm", "mask", "tp1"]
    for c in cases:
        globals()[f"case_{c}"]()
