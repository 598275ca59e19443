"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz).

CPU-only: these run in the build container and on any box without a GPU.
"""

import numpy as np
import pytest

from oracle import ffwd_oracle as orc
from tests.fixtures import golden, load_case

CASES_FFN = ["tiny_dfl", "tiny_all", "tiny_k25", "cfg1", "l1b"]
CASES_PRED = ["l8b_pred", "qwen8b_pred"]


def test_topk_edges_match_reference():
    g = golden("topk_edges")
    for i, k in enumerate(g["k"]):
        s = g["scores"][g["offs_s"][i]:g["offs_s"][i + 1]]
        want = g["indices"][g["offs_i"][i]:g["offs_i"][i + 1]]
        got = orc.topk_indices(s, int(k))
        np.testing.assert_array_equal(got, want, err_msg=f"case {i} k={k} s={s[:8]}")


def test_scheduler_matches_reference():
    g = golden("scheduler")
    offs = g["offs"]
    for i, budget in enumerate(g["budget"]):
        s = g["s"][offs[i]:offs[i + 1]]
        want = g["b"][offs[i]:offs[i + 1]]
        got = orc.allocate_budgets(s, float(budget))
        np.testing.assert_array_equal(got, want)
    for i, b in enumerate(g["k_budgets"]):
        for j, f in enumerate(g["k_dffn"]):
            assert orc.budget_to_k(float(b), int(f)) == g["k_out"][i, j]


@pytest.mark.parametrize("name", CASES_FFN + CASES_PRED)
def test_predictor_and_topk_bit_exact(name):
    c = load_case(name)
    p = c["pred"]
    for row, j in enumerate(c["sparse_blocks"]):
        lo, hi = int(j) * 128, min(c["T"], (int(j) + 1) * 128)
        s = orc.predictor_forward(p["query"], p["w1"], p["w2"], c["x"][lo:hi])
        np.testing.assert_array_equal(s.view(np.uint32), c["scores"][row].view(np.uint32))
        np.testing.assert_array_equal(orc.topk_indices(s, c["k"]), c["indices"][row])


@pytest.mark.parametrize("name", ["tiny_dfl", "tiny_all", "tiny_k25", "cfg1"])
def test_ffn_layer_matches_reference(name):
    c = load_case(name)
    y, masks, _ = orc.ffn_layer_blockwise(c["x"], c["lw"], c["pred"], c["comp"], c["k"],
                                          c["dense_first_last"], keep_masks=True)
    want = c["y"]
    got = y[c["y_rows"]] if "y_rows" in c else y
    # same algorithm, same f64-accumulate/f32-round points: equal up to the
    # f64 summation order of the BLAS underneath (invisible after rounding)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-6)
    assert abs(y.astype(np.float64).sum() - float(c["y_sum"])) < 1e-3
    for row, j in enumerate(c["sparse_blocks"]):
        np.testing.assert_array_equal(masks[int(j)], c["indices"][row])


def test_bf16_round_is_rne():
    v = np.array([1.0, 1.00390625, 1.005859375, 1.0019531, -2.5, np.inf, -np.inf, 0.0, -0.0,
                  3.3895314e38], np.float32)
    got = orc.bf16_round(v)
    import torch
    want = torch.from_numpy(v).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.isnan(orc.bf16_round(np.array([np.nan], np.float32)))[0]


def test_flop_definition_matches_reference_numbers():
    # per-layer algorithmic FLOPs at the 8B/16K config
    fl = orc.layer_flops(16384, 4096, 14336, 7168)
    assert fl["ffn"] + fl["predictor"] + fl["compensator"] == pytest.approx(3.0681e12, rel=1e-4)
    fl1 = orc.layer_flops(1024, 512, 1376, 688)
    assert sum(fl1.values()) == pytest.approx(2.8083e9, rel=1e-4)
