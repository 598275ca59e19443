"""CPU checks of the full-prefill (TTFT) path's host side against the reference's golden run."""

import numpy as np

from tests.fixtures import load_prefill_case


def test_prefill_inputs_regenerate_bit_exact():
    c = load_prefill_case()  # raises unless every weight digest matches the reference's
    g = c["golden"]
    assert g["masks"].shape == (len(g["mask_keys"]), int(g["k"]))
    for row in g["masks"]:
        assert (np.diff(row) > 0).all()


def test_prefill_flop_report_matches_reference():
    from paper_2602_00397_b200 import predict_prefill_flops
    c = load_prefill_case()
    g = c["golden"]
    L, d, f, V, T = (int(g[k]) for k in ("n_layers", "d", "f", "vocab", "T"))
    rep = predict_prefill_flops(L, d, f, V, T, b=[float(g["budget"])] * L,
                                dense_first_last=True, mode="predicted", has_compensators=True)
    assert rep.total() == int(g["flops_total"])


def test_model_weights_validation():
    import pytest
    from paper_2602_00397_b200.errors import ValidationError
    from paper_2602_00397_b200.model import LayerWeights, ModelConfig, ModelWeights
    c = load_prefill_case()
    g, m = c["golden"], c["model"]
    cfg = ModelConfig(n_layers=int(g["n_layers"]), d_model=int(g["d"]), d_ffn=int(g["f"]),
                      n_heads=int(g["n_heads"]), vocab_size=int(g["vocab"]),
                      max_context=int(g["T"]))
    layers = [LayerWeights(**lw) for lw in m["layers"]]
    w = ModelWeights(config=cfg, tok_emb=m["tok_emb"], layers=layers,
                     final_norm=m["final_norm"], w_out=m["w_out"])
    w.validate()
    assert w.out_head() is m["w_out"]
    bad = ModelWeights(config=cfg, tok_emb=m["tok_emb"][:, :8], layers=layers,
                       final_norm=m["final_norm"])
    with pytest.raises(ValidationError):
        bad.validate()


def test_prefill_flop_report_ablation_modes():
    from paper_2602_00397_b200 import predict_prefill_flops
    c = load_prefill_case()
    g = c["golden"]
    L, d, f, V, T = (int(g[k]) for k in ("n_layers", "d", "f", "vocab", "T"))
    for mode in ("oracle", "static"):
        rep = predict_prefill_flops(L, d, f, V, T, b=[float(g["budget"])] * L,
                                    dense_first_last=True, mode=mode, has_compensators=True)
        assert rep.total() == int(g[f"{mode}_flops_total"]), mode


def test_first_block_static_contract():
    import pytest
    from paper_2602_00397_b200 import ExpertMask, FirstBlockStatic
    from paper_2602_00397_b200.errors import ValidationError
    bank = FirstBlockStatic()
    with pytest.raises(ValidationError):
        bank.mask_for(0)
    m = ExpertMask(bits=np.array([0, 1, 1, 0], np.uint8), k=2, layer=3, block=0)
    bank.set_first(3, m)
    assert bank.mask_for(3) is m
