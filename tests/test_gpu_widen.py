"""The INT-pipe widening of bf16 / f32 operands to f64 (csrc/widen.cuh) in the pooling
pass and the FFN-input RMSNorm must give exactly the F2F results: inputs holding exact
zeros, bf16 / f32 subnormals and huge values (warps that fall back to F2F next to warps
that do not) still produce the oracle's predictor scores bit for bit and the reference
RMSNorm's output."""

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


def test_pooling_with_special_values_bit_exact(ff):
    from paper_2602_00397_b200.predictor import predictor_scores
    d, f, T = 1024, 2048, 8 * 128
    rng = np.random.default_rng(17)
    x = rng.standard_normal((T, d)).astype(np.float32)
    x[128:256, ::7] = 0.0                               # exact zeros in block 1
    x[256:384, 5] = np.float32(3e-39)                   # subnormal in block 2
    x[384:512, 100:108] = np.float32(-1.5e-39)
    x[512:640, 9] = np.float32(1e30)                    # huge but finite (block 4)
    x = orc.bf16_round(x)
    pred = orc.init_predictor(np.random.default_rng(3), d, f)
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    got = predictor_scores(dp, torch.from_numpy(x).cuda().to(torch.bfloat16)).cpu().numpy()
    for b in range(T // 128):
        want = orc.predictor_forward(pred["query"], pred["w1"], pred["w2"],
                                     x[b * 128:(b + 1) * 128])
        assert np.array_equal(got[b], want), f"block {b}"


def test_rmsnorm_with_special_values(ff):
    from paper_2602_00397_b200.norm import rmsnorm
    from paper_2602_00397_b200.predictor import predictor_logits
    T, d = 64, 2048
    rng = np.random.default_rng(5)
    x = rng.standard_normal((T, d)).astype(np.float32)
    x[3, ::3] = 0.0
    x[7, 11] = np.float32(1e-40)   # f32 subnormal
    x[9, :] = 0.0
    x[9, 0] = 1.0
    x[12, 200:300] = np.float32(3e-39)
    gain = np.ones(d, np.float32)
    pred = orc.init_predictor(np.random.default_rng(6), d, 256)
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    xb, x32, lg = rmsnorm(torch.from_numpy(x).cuda(), torch.from_numpy(gain).cuda(),
                          out_f32=True, predictor=dp)
    x64 = x.astype(np.float64)
    want = (x64 / np.sqrt((x64 * x64).mean(axis=1, keepdims=True) + 1e-6)).astype(np.float32)
    got = x32.cpu().numpy()
    diff = got != want
    assert diff.mean() <= 1e-4
    if diff.any():
        assert np.abs(got[diff].view(np.int32).astype(np.int64)
                      - want[diff].view(np.int32).astype(np.int64)).max() <= 1
    assert torch.equal(lg, predictor_logits(dp, xb))
