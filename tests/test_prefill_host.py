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
