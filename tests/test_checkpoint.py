"""`.ffwd` checkpoints: the native reader against files written by the REFERENCE's own
writer (tests/golden/tiny_*.ffwd, make_golden.make_checkpoint_case), byte-identical
writing, and the reference's validation errors (checkpoint.py:207-263)."""

import os
import struct

import numpy as np
import pytest

from oracle import ffwd_oracle as orc
from tests.fixtures import GOLDEN

SEED, L, D, F, H, V = 77, 2, 64, 160, 2, 50


@pytest.fixture(scope="module")
def ck():
    from paper_2602_00397_b200 import checkpoint
    return checkpoint


def _expected():
    m = orc.synthetic_model(SEED, L, D, F, V)
    preds = [orc.init_predictor(np.random.default_rng([SEED, l]), D, F) for l in range(L)]
    comps = [orc.init_compensator(np.random.default_rng([SEED + 1, l]), D) for l in range(L)]
    return m, preds, comps


def test_reads_reference_written_files(ck):
    m, preds, comps = _expected()
    c = ck.read_checkpoint(os.path.join(GOLDEN, "tiny_model.ffwd"))
    assert c.config.to_json_dict() == {"n_layers": L, "d_model": D, "d_ffn": F, "n_heads": H,
                                       "vocab_size": V, "block_size": 128, "max_context": 256}
    assert np.array_equal(c.weights.tok_emb, m["tok_emb"])
    assert np.array_equal(c.weights.w_out, m["w_out"])
    for lw, ref in zip(c.weights.layers, m["layers"]):
        for name in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down", "attn_norm",
                     "ffn_norm"):
            assert np.array_equal(getattr(lw, name), ref[name]), name
    assert c.predictors is None and c.compensators is None
    a = ck.read_checkpoint(os.path.join(GOLDEN, "tiny_aux.ffwd"))
    assert a.weights is None
    for p, ref in zip(a.predictors, preds):
        assert np.array_equal(p.query, ref["query"]) and np.array_equal(p.w2, ref["w2"])
    for cc, ref in zip(a.compensators, comps):
        assert np.array_equal(cc.w1, ref["w1"]) and np.array_equal(cc.w2, ref["w2"])


def test_writer_is_byte_identical_to_reference(ck, tmp_path):
    c = ck.read_checkpoint(os.path.join(GOLDEN, "tiny_model.ffwd"))
    a = ck.read_checkpoint(os.path.join(GOLDEN, "tiny_aux.ffwd"))
    ck.write_checkpoint(tmp_path / "m.ffwd", c.config, weights=c.weights)
    ck.write_checkpoint(tmp_path / "a.ffwd", a.config, predictors=a.predictors,
                        compensators=a.compensators)
    for mine, ref in (("m.ffwd", "tiny_model.ffwd"), ("a.ffwd", "tiny_aux.ffwd")):
        assert (tmp_path / mine).read_bytes() == open(os.path.join(GOLDEN, ref), "rb").read()


def _corrupt(tmp_path, name, blob):
    p = tmp_path / name
    p.write_bytes(blob)
    return p


def test_validation_errors_match_reference(ck, tmp_path):
    from paper_2602_00397_b200.errors import ValidationError
    good = open(os.path.join(GOLDEN, "tiny_aux.ffwd"), "rb").read()
    cases = {
        "magic": (b"NOPE" + good[4:], "is not an engine checkpoint"),
        "version": (good[:4] + struct.pack("<I", 2) + good[8:], "unsupported checkpoint version"),
        "truncated": (good[:len(good) // 2], "truncated while reading"),
        "empty": (b"", "truncated while reading magic"),
    }
    # dtype of the first tensor: directory starts after magic, version, config
    clen = struct.unpack("<I", good[8:12])[0]
    p0 = 12 + clen + 4
    nl = struct.unpack("<H", good[p0:p0 + 2])[0]
    dpos = p0 + 2 + nl
    cases["dtype"] = (good[:dpos] + b"f16 " + good[dpos + 4:], "unsupported dtype")
    for name, (blob, msg) in cases.items():
        with pytest.raises(ValidationError, match=msg):
            ck.read_checkpoint(_corrupt(tmp_path, name + ".ffwd", blob))


def test_config_json_roundtrip_and_load_model_warning(ck, tmp_path):
    import warnings
    from paper_2602_00397_b200.model import ModelConfig
    c = ck.read_checkpoint(os.path.join(GOLDEN, "tiny_model.ffwd"))
    ck.save_config_json(c.config, tmp_path / "cfg.json")
    assert ck.load_config_json(tmp_path / "cfg.json").to_json_dict() == c.config.to_json_dict()
    other = ModelConfig(n_layers=L, d_model=D, d_ffn=F, n_heads=H, vocab_size=V + 1)
    ck.save_config_json(other, tmp_path / "other.json")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        wts = ck.load_model(os.path.join(GOLDEN, "tiny_model.ffwd"), tmp_path / "other.json")
    assert any("disagrees" in str(x.message) for x in w)
    assert wts.config.vocab_size == V
