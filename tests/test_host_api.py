"""Host-side logic of the drop-in API (no GPU): scheduler, plans, masks,
sharding, FLOP accounting -- checked against the reference's golden vectors
and the reference's own test expectations (test_scheduler.py, test_sparse.py,
test_costmodel.py)."""

import json

import numpy as np
import pytest

import paper_2602_00397_b200 as ff
from oracle import ffwd_oracle as orc
from tests.fixtures import golden


def test_allocate_budgets_matches_reference_bitwise():
    g = golden("scheduler")
    offs = g["offs"]
    for i, budget in enumerate(g["budget"]):
        s = g["s"][offs[i]:offs[i + 1]]
        np.testing.assert_array_equal(ff.allocate_budgets(s, float(budget)),
                                      g["b"][offs[i]:offs[i + 1]])


def test_allocate_budgets_hand_traces():
    # scheduler.py:66-93 traces (reference test_scheduler.py:23-46)
    np.testing.assert_allclose(ff.allocate_budgets([4.0, 2.0, 1.0, 1.0], 0.5),
                               [1.0, 0.5, 0.25, 0.25], atol=1e-12)
    np.testing.assert_allclose(ff.allocate_budgets([1.0, 4.0], 0.9), [0.36, 1.0], atol=1e-12)
    b = ff.allocate_budgets([1.0, 1.0, 100.0], 0.9)
    assert b[2] == 1.0 and b.sum() < 0.9 * 3  # a late cap leaks budget on purpose
    for bad in (([1.0, 2.0], 0.0), ([1.0, 2.0], 1.5), ([1.0, -2.0], 0.5), ([0.0, 0.0], 0.5),
                ([], 0.5)):
        with pytest.raises(ff.ValidationError):
            ff.allocate_budgets(*bad)


def test_budget_to_k_matches_reference():
    g = golden("scheduler")
    for i, b in enumerate(g["k_budgets"]):
        for j, f in enumerate(g["k_dffn"]):
            assert ff.budget_to_k(float(b), int(f)) == g["k_out"][i, j]
    assert ff.budgets_to_topk([1.0, 0.5, 0.004], 64) == [64, 32, 1]
    with pytest.raises(ff.ValidationError):
        ff.budget_to_k(0.0, 10)


def test_sparsity_plan_roundtrip_and_validation(tmp_path):
    plan = ff.plan_from_profile(ff.AttentionMassProfile(s=np.array([3.0, 1.0, 2.0, 2.0]),
                                                        n_sequences=2, n_heads=4), 0.5, seed=7,
                                calibration="synthetic")
    p = tmp_path / "plan.json"
    ff.save_plan(plan, p)
    back = ff.load_plan(p)
    np.testing.assert_array_equal(back.b, plan.b)
    assert back.dense_first_last and back.seed == 7
    assert back.ks(14336) == [ff.budget_to_k(float(b), 14336) for b in plan.b]
    assert json.loads(p.read_text())["calibration"] == "synthetic"
    with pytest.raises(ff.ValidationError):
        ff.SparsityPlan(b=np.array([0.9, 0.9]), dense_first_last=True, budget=0.5)
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(ff.ValidationError):
        ff.load_plan(tmp_path / "bad.json")
    assert ff.uniform_plan(3, 0.5).ks(100) == [50, 50, 50]
    assert ff.dense_plan(2).ks(100) == [100, 100]


def test_expert_mask_validation():
    m = ff.ExpertMask(bits=np.array([0, 1, 1, 0, 1], np.uint8), k=3)
    np.testing.assert_array_equal(m.indices, [1, 2, 4])
    with pytest.raises(ff.ValidationError):
        ff.ExpertMask(bits=np.array([0, 1, 1], np.uint8), k=3)
    with pytest.raises(ff.ValidationError):
        ff.ExpertMask(bits=np.array([0, 2, 1], np.uint8), k=3)
    lw = ff.LayerWeights(w_gate=np.zeros((4, 5), np.float32), w_up=np.zeros((4, 5), np.float32),
                         w_down=np.zeros((5, 4), np.float32))
    with pytest.raises(ff.ValidationError):
        ff.select_subweights(lw, ff.ExpertMask(bits=np.array([1, 0, 0, 1], np.uint8), k=2))
    sub = ff.select_subweights(lw, ff.ExpertMask(bits=np.array([1, 0, 0, 1, 0], np.uint8), k=2))
    assert sub.w_gate.shape == (4, 2) and sub.w_down.shape == (2, 4)


def test_model_config_contract():
    cfg = ff.ModelConfig(n_layers=32, d_model=4096, d_ffn=14336, n_heads=32, vocab_size=128,
                         max_context=16384)
    assert cfg.n_blocks(16384) == 128 and cfg.n_blocks(300) == 3
    assert ff.ModelConfig.from_json_dict(cfg.to_json_dict()) == cfg
    with pytest.raises(ff.ValidationError):
        ff.ModelConfig(n_layers=1, d_model=64, d_ffn=32, n_heads=1, vocab_size=4)
    assert ff.default_reduced_dim(4096) == 256 and ff.default_reduced_dim(3072) == 256
    assert ff.default_comp_dim(4096) == 512 and ff.default_comp_dim(4) == 1


@pytest.mark.parametrize("tp", [1, 2, 3, 4, 8])
def test_neuron_and_compensator_shards_partition(tp):
    f, rc = 14336, 512
    ids = np.concatenate([ff.shard_neurons(f, r, tp) for r in range(tp)])
    assert np.array_equal(np.sort(ids), np.arange(f))
    spans = [ff.shard_comp_cols(rc, r, tp) for r in range(tp)]
    assert spans[0][0] == 0 and spans[-1][1] == rc
    assert all(spans[i][1] == spans[i + 1][0] for i in range(tp - 1))
    with pytest.raises(ff.ValidationError):
        ff.shard_neurons(f, tp, tp)


def test_flop_accounting_matches_reference_numbers():
    # SURVEY 8(d) / BASELINE.md: algorithmic FLOPs per layer (costmodel.py:108-177)
    assert ff.ffn_path_flops(4096, 14336, 16384, 7168) == pytest.approx(3.0681e12, rel=1e-4)
    assert ff.ffn_path_flops(2048, 8192, 4096, 4096) == pytest.approx(2.2721e11, rel=1e-4)
    assert ff.ffn_path_flops(512, 1376, 1024, 688) == pytest.approx(2.8083e9, rel=1e-4)
    for d, f, T, k in [(512, 1376, 1024, 688), (128, 384, 300, 192), (4096, 14336, 16384, 7168)]:
        fl = orc.layer_flops(T, d, f, k)
        assert ff.ffn_path_flops(d, f, T, k) == sum(fl.values())
    rep = ff.predict_prefill_flops(32, 4096, 14336, 128256, 4096, b=[0.5] * 32,
                                   dense_first_last=True, mode="predicted", has_compensators=True)
    dense = ff.predict_prefill_flops(32, 4096, 14336, 128256, 4096)
    # the reference's analytic 8B/4K speedup (1.4319) -- vocab does not move it
    assert dense.total() / rep.total() == pytest.approx(1.4319, abs=2e-3)
