"""Parity of the exact path `bench.py` times, at every BASELINE configuration.

The bench's step per layer (engine.py:267-308): the FFN-input RMSNorm of the f32
residual stream fused with the predictor's per-token logits (``norm.rmsnorm(...,
predictor=...)``) -> ``sparse_ffn_layer(..., logits_in=...)`` with the residual add
fused into the down projection.  This test runs that sequence layer after layer
(each layer's input is the previous layer's GPU output) and checks, at full size:

  * every predicted block's index row equals the oracle's top-k of the oracle's
    predictor scores on the same FFN input (``np.array_equal``; predictor.py:68-81,
    kernels.py:139-149, engine.py:284-288) -- all blocks, not a sample;
  * the fused logits change nothing: the same layer run without ``logits_in`` (the
    predictor's own first pooling pass) gives bit-identical indices and outputs;
  * at least 8 blocks per layer (the dense first and last, 6 predicted) are within the
    parity tolerance of the oracle's FFN (+ compensator) output: rel-L2 <= 5e-3,
    max|d| <= 3e-2 rms(y_ref).

Both predictor input modes are covered: ``bf16`` (the bench's headline: the predictor
pools the bf16 FFN operand) and ``f32`` (the reference's own predictor input, the f32
RMSNorm output, engine.py:267,286: ``logits_from_f32`` + ``x_pred_f32``).

Configurations (BASELINE.json configs[1..4]): Llama-3.1-8B shape at T=16384 with 50%,
25% and 75% keep; Qwen3-8B shape at T=8192 with per-layer k from the layer-wise
schedule (``allocate_budgets``, scheduler.py:66-98; four layers of different k); the
Llama-3.2-1B shape at T=4096.
"""

import numpy as np
import pytest
import torch

from oracle import ffwd_oracle as orc

pytestmark = pytest.mark.gpu

REL_L2 = 5e-3
MAX_REL_RMS = 3e-2


@pytest.fixture(scope="module")
def ff():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_00397_b200 as ff
    from paper_2602_00397_b200 import _lib
    _lib.require_device(torch.cuda.current_device())
    return ff


def qwen_schedule(f: int, L: int = 36, budget: float = 0.5, seed: int = 1234):
    """bench.py's Qwen3 schedule: a seeded importance profile through Algorithm 1."""
    s = np.random.default_rng(seed).random(L) + 0.25
    b = orc.allocate_budgets(s, budget)
    return [orc.budget_to_k(float(v), f) for v in b]


def pick_distinct(ks, n=4):
    """n layer ids whose k values are distinct and spread over the schedule's range
    (the smallest, the largest and evenly spaced ranks between)."""
    order = sorted(range(len(ks)), key=lambda i: (ks[i], i))
    picks = [order[int(p)] for p in np.linspace(0, len(order) - 1, n).round()]
    assert len({ks[i] for i in picks}) == n
    return sorted(picks)


CASES = {
    # name: (d, f, T, [(layer seed, k)], predictor modes)
    "8b_k50": (4096, 14336, 16384, [(0, orc.budget_to_k(0.5, 14336))], ("bf16", "f32")),
    "8b_k25": (4096, 14336, 16384, [(1, orc.budget_to_k(0.25, 14336))], ("bf16",)),
    "8b_k75": (4096, 14336, 16384, [(2, orc.budget_to_k(0.75, 14336))], ("bf16",)),
    "1b": (2048, 8192, 4096, [(0, 4096), (1, 4096)], ("bf16", "f32")),
}


def _qwen_case():
    ks = qwen_schedule(12288)
    layers = pick_distinct(ks)
    return (4096, 12288, 8192, [(l, ks[l]) for l in layers], ("bf16",))


def make_layer(ff, d, f, seed):
    rng = np.random.default_rng([2026, seed])
    lw = {n: orc.bf16_round((rng.standard_normal(shape, dtype=np.float32) * np.float32(0.02)))
          for n, shape in (("w_gate", (d, f)), ("w_up", (d, f)), ("w_down", (f, d)))}
    pred = orc.init_predictor(np.random.default_rng([2026, seed, 1]), d, f)
    comp = {k: orc.bf16_round(v) for k, v in
            orc.init_compensator(np.random.default_rng([2026, seed, 2]), d).items()}
    packed = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], ff.CompensatorParams(**comp),
                           device="cuda")
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    return lw, pred, comp, packed, dp


def assert_close(got, want, what):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    rms = np.sqrt((want ** 2).mean())
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    mx = np.abs(got - want).max() / max(rms, 1e-30)
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    assert rel <= REL_L2, f"{what}: rel-L2 {rel:.3e} > {REL_L2}"
    assert mx <= MAX_REL_RMS, f"{what}: max|d|/rms {mx:.3e} > {MAX_REL_RMS}"


@pytest.mark.parametrize("name", ["8b_k50", "8b_k25", "8b_k75", "qwen8b", "1b"])
def test_timed_path_indices_bit_exact_every_block(ff, name):
    from paper_2602_00397_b200.norm import rmsnorm
    d, f, T, layers, modes = _qwen_case() if name == "qwen8b" else CASES[name]
    n_blk = T // 128
    gain = torch.ones(d, device="cuda")  # ffn_norm gains (synthetic.py:41)
    for mode in modes:
        res = torch.randn((T, d), generator=torch.Generator().manual_seed(99)).to(
            torch.bfloat16).float().cuda()
        xb = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
        x32 = torch.empty((T, d), dtype=torch.float32, device="cuda") if mode == "f32" else None
        lg = torch.empty((T,), dtype=torch.float32, device="cuda")
        for seed, k in layers:
            lw, pred, comp, packed, dp = make_layer(ff, d, f, seed)
            before = res.clone()
            rmsnorm(res, gain, out=xb, out_f32=mode == "f32", out32=x32, predictor=dp, logits=lg,
                    logits_from_f32=mode == "f32")
            xp = x32 if mode == "f32" else None
            # the bench's call: fused logits, residual add in the K3 epilogue, in place
            _, idx = ff.sparse_ffn_layer(xb, packed, dp, k, out=res, residual=res, logits_in=lg,
                                         x_pred_f32=xp, return_indices=True)
            # the same layer through the predictor's own first pass (no fused logits)
            alt = before.clone()
            _, idx2 = ff.sparse_ffn_layer(xb, packed, dp, k, out=alt, residual=alt,
                                          x_pred_f32=xp, return_indices=True)
            torch.cuda.synchronize()
            tag = f"{name} {mode} layer {seed} k={k}"
            assert torch.equal(idx, idx2), f"{tag}: fused logits changed the selection"
            assert torch.equal(res, alt), f"{tag}: fused logits changed the output"
            x_in = (x32 if mode == "f32" else xb).float().cpu().numpy()
            x_ffn = xb.float().cpu().numpy()
            got = idx.cpu().numpy()
            assert got.shape == (n_blk - 2, k)
            for j in range(1, n_blk - 1):  # every predicted block (dense first/last)
                s = orc.predictor_forward(pred["query"], pred["w1"], pred["w2"],
                                          x_in[j * 128:(j + 1) * 128])
                want = orc.topk_indices(s, k)
                if not np.array_equal(got[j - 1], want):
                    bad = np.setxor1d(got[j - 1], want)
                    raise AssertionError(f"{tag}: block {j} indices differ from the oracle "
                                         f"({bad.size} neurons: {bad[:8]})")
            y = (res - before).cpu().numpy()
            check = sorted({0, n_blk - 1, 1, n_blk - 2} |
                           set(np.linspace(2, n_blk - 3, 4).round().astype(int).tolist()))
            assert len(check) >= 8
            for j in check:
                xs = x_ffn[j * 128:(j + 1) * 128]
                if j in (0, n_blk - 1):
                    want_y = orc.dense_ffn(xs, lw["w_gate"], lw["w_up"], lw["w_down"])
                else:
                    want_y = orc.sparse_ffn_forward(xs, lw["w_gate"], lw["w_up"], lw["w_down"],
                                                    got[j - 1])
                    want_y = want_y + orc.compensator_forward(comp["w1"], comp["w2"], xs)
                assert_close(y[j * 128:(j + 1) * 128], want_y, f"{tag} block {j}")
            del packed, dp
            torch.cuda.empty_cache()
