"""Analytic FLOP accounting (``costmodel.py:24-193``): the algorithmic-FLOP
definition behind every effective-TFLOP/s and roofline number of this build.

GPU work bypasses the reference's instrumented ``kernels.matmul`` counter, so
the report is charged analytically with exactly the reference's formulas:
FFN ``6 n d k`` (``:171``), predictor ``4 n d + 2 d r + 2 r f`` (``:170``),
compensator ``4 n d r'`` (``:175``), dense ``6 n d f`` (``:163``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .compensator import default_comp_dim
from .errors import ValidationError
from .predictor import default_reduced_dim
from .sparse import budget_to_k

LAYER_COMPONENTS = ("attn_proj", "attn_scores", "ffn", "predictor", "compensator")
MODES = ("dense", "oracle", "predicted", "static")


@dataclass
class FlopsReport:
    n_tokens: int
    mode: str
    per_layer: list = field(default_factory=list)
    output_head: int = 0

    @classmethod
    def empty(cls, n_layers: int, n_tokens: int, mode: str) -> "FlopsReport":
        return cls(n_tokens=n_tokens, mode=mode,
                   per_layer=[{c: 0 for c in LAYER_COMPONENTS} for _ in range(n_layers)])

    def add(self, layer: int, component: str, flops: int) -> None:
        self.per_layer[layer][component] += flops

    def component_totals(self) -> dict:
        totals = {c: sum(l[c] for l in self.per_layer) for c in LAYER_COMPONENTS}
        totals["output_head"] = self.output_head
        return totals

    def total(self) -> int:
        return sum(self.component_totals().values())

    def to_dict(self) -> dict:
        return {"n_tokens": self.n_tokens, "mode": self.mode,
                "per_layer": [dict(l) for l in self.per_layer], "output_head": self.output_head,
                "component_totals": self.component_totals(), "total": self.total()}


def predict_prefill_flops(n_layers: int, d_model: int, d_ffn: int, vocab_size: int, T: int,
                          b=None, dense_first_last: bool = False, mode: str = "dense",
                          has_compensators: bool = False, include_predictor: bool = True,
                          predictor_r: int | None = None, compensator_r: int | None = None,
                          block_size: int = 128) -> FlopsReport:
    """Analytic twin of the block-wise prefill FLOP report (``costmodel.py:108-177``)."""
    if mode not in MODES:
        raise ValidationError(f"unknown mode {mode!r}")
    if T < 1:
        raise ValidationError("T must be >= 1")
    if mode == "dense":
        ks, dfl = None, False
    else:
        if b is None or len(b) != n_layers:
            raise ValidationError(f"mode {mode!r} requires one keep fraction per layer")
        ks = [budget_to_k(float(x), d_ffn) for x in b]
        dfl = bool(dense_first_last)
    d, f = d_model, d_ffn
    r = default_reduced_dim(d) if predictor_r is None else predictor_r
    rc = default_comp_dim(d) if compensator_r is None else compensator_r
    rep = FlopsReport.empty(n_layers, T, mode)
    spans = [(lo, min(T, lo + block_size)) for lo in range(0, T, block_size)]
    cache_len = 0
    for j, (lo, hi) in enumerate(spans):
        n = hi - lo
        cache_len += n
        dense_block = mode == "dense" or (dfl and j in (0, len(spans) - 1)) or \
            (mode == "static" and j == 0)
        for l in range(n_layers):
            rep.add(l, "attn_proj", 8 * n * d * d)
            rep.add(l, "attn_scores", 4 * n * cache_len * d)
            if dense_block or (ks is not None and ks[l] == f):
                rep.add(l, "ffn", 6 * n * d * f)
                continue
            k = ks[l]
            if mode == "oracle":
                rep.add(l, "ffn", 4 * n * d * f + 6 * n * d * k)
            elif mode == "predicted":
                if include_predictor:
                    rep.add(l, "predictor", 4 * n * d + 2 * d * r + 2 * r * f)
                rep.add(l, "ffn", 6 * n * d * k)
            else:
                rep.add(l, "ffn", 6 * n * d * k)
            if has_compensators:
                rep.add(l, "compensator", 4 * n * d * rc)
    rep.output_head = 2 * d * vocab_size
    return rep


def ffn_path_flops(d: int, f: int, T: int, k: int, dense_first_last: bool = True,
                   has_comp: bool = True, block_size: int = 128) -> int:
    """Algorithmic FLOPs of one layer's FFN hot path: ffn + predictor + compensator,
    charged per block exactly as ``costmodel.py:159-175`` (k given directly)."""
    r, rc = default_reduced_dim(d), default_comp_dim(d)
    spans = [(lo, min(T, lo + block_size)) for lo in range(0, T, block_size)]
    tot = 0
    for j, (lo, hi) in enumerate(spans):
        n = hi - lo
        if k >= f or (dense_first_last and j in (0, len(spans) - 1)):
            tot += 6 * n * d * f
        else:
            tot += 6 * n * d * k + 4 * n * d + 2 * d * r + 2 * r * f
            if has_comp:
                tot += 4 * n * d * rc
    return tot


def dense_ffn_flops(d: int, f: int, T: int) -> int:
    return 6 * T * d * f
