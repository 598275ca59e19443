"""Shared test fixtures: regenerate the golden cases' weights with the oracle.

The golden ``.npz`` files hold the reference's outputs plus SHA-256 digests
of the weights the reference saw; ``load_case`` regenerates those weights
with the oracle's generators (same seeds, same draw order) and refuses to
continue if a digest differs, so every consumer is provably fed the exact
inputs the reference was.
"""

from __future__ import annotations

import hashlib
import os

import numpy as np

from oracle import ffwd_oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def make_inputs(d, f, T, seed, layer=0, with_ffn=True):
    """Oracle-side regeneration of make_golden.make_case's inputs."""
    pred = orc.init_predictor(np.random.default_rng([seed, layer]), d, f)
    comp = orc.init_compensator(np.random.default_rng([seed + 1, layer]), d)
    comp = {k: orc.bf16_round(v) for k, v in comp.items()}
    x = orc.bf16_round(np.random.default_rng([seed, layer, 99]).standard_normal((T, d))
                       .astype(np.float32))
    lw = None
    if with_ffn:
        lw = orc.random_layer(np.random.default_rng([seed, layer, 7]), d, f, 0.02)
        lw = {k: (orc.bf16_round(v) if k in ("w_gate", "w_up", "w_down") else v)
              for k, v in lw.items()}
    return x, lw, pred, comp


def load_case(name: str, check_sha: bool = True) -> dict:
    g = golden(name)
    d, f, T, seed, layer = (int(g[k]) for k in ("d", "f", "T", "seed", "layer"))
    with_ffn = "sha_ffn" in g
    x, lw, pred, comp = make_inputs(d, f, T, seed, layer, with_ffn)
    if check_sha:
        assert sha(x) == str(g["sha_x"]), f"{name}: regenerated x differs from the reference's"
        assert sha(pred["query"], pred["w1"], pred["w2"]) == str(g["sha_pred"])
        assert sha(comp["w1"], comp["w2"]) == str(g["sha_comp"])
        if with_ffn:
            assert sha(lw["w_gate"], lw["w_up"], lw["w_down"]) == str(g["sha_ffn"])
    g.update(x=x, lw=lw, pred=pred, comp=comp, d=d, f=f, T=T, k=int(g["k"]),
             dense_first_last=bool(int(g["dense_first_last"])))
    return g


def load_prefill_case(name: str = "prefill_small") -> dict:
    """Regenerate the golden full-prefill case (make_golden.make_prefill_case) with the
    oracle and check every input against the reference's digests."""
    g = golden(name)
    seed, L, d, f, V, T = (int(g[k]) for k in ("seed", "n_layers", "d", "f", "vocab", "T"))
    m = orc.synthetic_model(seed, L, d, f, V)
    for lw in m["layers"]:
        for kk in ("w_gate", "w_up", "w_down"):
            lw[kk] = orc.bf16_round(lw[kk])
    preds = [orc.init_predictor(np.random.default_rng([seed, l]), d, f) for l in range(L)]
    comps = [{k: orc.bf16_round(v) for k, v in
              orc.init_compensator(np.random.default_rng([seed + 1, l]), d).items()}
             for l in range(L)]
    tokens = np.random.default_rng([seed, 5]).integers(0, V, T)
    digests = {
        "sha_model": sha(m["tok_emb"], m["w_out"], *[lw[n] for lw in m["layers"] for n in
                                                      ("wq", "wk", "wv", "wo", "w_gate", "w_up",
                                                       "w_down")]),
        "sha_pred": sha(*[a for p in preds for a in (p["query"], p["w1"], p["w2"])]),
        "sha_comp": sha(*[a for c in comps for a in (c["w1"], c["w2"])]),
        "sha_tokens": sha(tokens),
    }
    for k, v in digests.items():
        if str(g[k]) != v:
            raise AssertionError(f"{name}: regenerated {k} differs from the reference's inputs")
    return dict(golden=g, model=m, preds=preds, comps=comps, tokens=tokens)
