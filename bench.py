#!/usr/bin/env python
"""Benchmark: FastForward prefill-FFN hot path on B200 (BASELINE.json metric).

Metric: "Llama-3.1-8B prefill FFN ms/layer & TTFT at 50% sparsity vs dense, 4K-16K".
Workload (N=1, BASELINE configs[2] at one GPU): Llama-3.1-8B FFN shape
(d_model 4096, d_ffn 14336, 32 layers), T = 16384 tokens, 128-token blocks,
50% keep (k = 7168), dense first/last block, predictor + compensator
(r 256, r' 512), random-init weights (normal x 0.02, synthetic.py:33-43).

One step = the prefill FFN stack: for each of the 32 layers (own weights, own
predictor and compensator) the FFN branch of engine.py:264-308 over all 128
blocks -- the FFN-input RMSNorm of the f32 residual stream (fused with the
predictor's per-token logits), predictor -> top-k -> sparse SwiGLU FFN +
compensator -> residual add.  The norm keeps the stack numerically sane (an
FFN-only stack without it overflows to inf by layer 6).  `value` = device time
per step / 32 (ms per layer), inputs resident in HBM, uninstrumented (the
per-kernel breakdown comes from a second, event-timed run); `e2e` = the same stack through the public API with the
prompt's hidden states copied from pinned host memory and the result copied
back inside the timed region, every step (the copies of step i+1 / i overlap step
i's compute on a copy stream, double-buffered).  Every input (X 128 MiB, weights 361 MiB per
layer) is larger than L2 and each layer has its own weights, so no L2 flush is
needed between iterations.

Under torchrun (N > 1), by default (`--parallel sp`): the prompt's 128-token
blocks are split into N contiguous shards, one per GPU, with the weights
replicated.  The FFN branch is block-local (engine.py:254-310: each block's
predictor, top-k, FFN and compensator see only that block), so no data-path
collective exists; only the ranks holding the prompt's first / last block run
it dense.  Scaling "strong" (one prompt, total work fixed).
`--parallel tp`: tensor parallel over d_ffn (strided neuron shards,
replicated predictor, sharded compensator) with one all-reduce of each layer's
output -- NCCL, or with `--collective fused` the peer-memory kernel that also
adds the residual (tp.PeerBuffers), or with `--collective overlap` that kernel
draining blocks while the down projection still runs (PeerBuffers.layer_overlap);
scaling "strong" (total work fixed).
`--parallel dp`: one prompt per GPU, no collective; scaling "weak".
The TTFT leg (N = 1) times the full 32-layer prefill (prefill.py) in the
predicted and dense modes.

`--impl reference` times the reference's own CPU implementation (the
unmodified `sparseprefill` package from baseline/_ref when present, else the
oracle port) on the host cores for a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "Llama-3.1-8B prefill FFN ms/layer & TTFT at 50% sparsity vs dense, 4K–16K"
CONFIGS = {
    # name: (d_model, d_ffn, n_layers, T, keep)
    "8b": (4096, 14336, 32, 16384, 0.5),
    "1b": (2048, 8192, 16, 4096, 0.5),
    "qwen8b": (4096, 12288, 36, 8192, 0.5),
    "cfg1": (512, 1376, 1, 1024, 0.5),
}
WORKLOAD_NAMES = {
    "8b": "Llama-3.1-8B-shape FFN stack (d4096 f14336 x32 layers), T=16384, 50% keep, "
          "predictor+compensator, dense first/last block",
    "1b": "Llama-3.2-1B-shape FFN stack (d2048 f8192 x16), T=4096, 50% keep",
    "qwen8b": "Qwen3-8B-shape FFN stack (d4096 f12288 x36), T=8192, layer-wise schedule, "
              "budget 0.5",
    "cfg1": "single SwiGLU FFN layer d512 f1376, T=1024, 50% keep",
}


def workload_config(args, T: int, L: int, ks, world: int) -> dict:
    """The workload both arms report (identical dicts: the driver compares them)."""
    d, f, _, _, keep = CONFIGS[args.config]
    par = args.parallel if world > 1 else "single"
    return {"workload": WORKLOAD_NAMES[args.config], "global_batch": 1 if par != "dp" else world,
            "seq_len": T, "layers": L, "keep": keep,
            "k_per_layer": list(ks) if args.config == "qwen8b" else ks[0], "block": 128,
            "dense_first_last": True, "parallelism": par if par == "single" else f"{par}{world}"}


def config_ks(cfg_name: str) -> list:
    """Per-layer k: budget_to_k(keep) everywhere, or the Qwen3 layer-wise schedule
    (a seeded importance profile through Algorithm 1, scheduler.py:66-98)."""
    import paper_2602_00397_b200 as ff  # host-side scheduler (scheduler.py mirror)
    d, f, L, T, keep = CONFIGS[cfg_name]
    if cfg_name == "qwen8b":
        s = np.random.default_rng(1234).random(L) + 0.25
        return [int(k) for k in ff.budgets_to_topk(ff.allocate_budgets(s, keep), f)]
    return [ff.budget_to_k(keep, f)] * L


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm": d.get("hbm_gbs", 6551.0), "bf16": d.get("bf16_tflops", 1639.5),
                "bf16_sus": d.get("bf16_tflops_sustained", 1376.2), "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback"}


# One process per GPU over NCCL.  FFWD_BENCH_BACKEND=gloo is a functional emulation for
# tests: every rank shares GPU 0 (time-sliced; numbers meaningless), which exercises the
# tensor-parallel path with the fused peer-memory completion (no NCCL data path) on one GPU.
BACKEND = os.environ.get("FFWD_BENCH_BACKEND", "nccl")


def local_device() -> int:
    return 0 if BACKEND == "gloo" else int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows: list[list[str]] = []
        self.times: list[float] = []  # arrival time of each row
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])
            self.times.append(time.monotonic())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0: float | None = None, t1: float | None = None) -> dict:
        """Rows that arrived inside [t0, t1 + 0.3 s] (the timed region; a row arrives shortly
        after its sample); a region shorter than the sampling period gets the first row
        after t0, flagged as "nearest"."""
        rows, note = self.rows, None
        if t0 is not None and t1 is not None:
            rows = [r for r, t in zip(self.rows, self.times) if t0 <= t <= t1 + 0.3]
            if not rows:
                after = [r for r, t in zip(self.rows, self.times) if t >= t0]
                rows, note = after[:1], "nearest sample after a timed region shorter than the sampling period"
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "power_w": None}
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except (ValueError, IndexError):
                continue
            try:
                pw.append(float(r[3]))
            except (ValueError, IndexError):
                pass
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        loaded = [v for v in sm if v > 0.5 * (mx or 1)] or sm
        out = {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm),
               "power_w": statistics.median(pw) if pw else None}
        if note:
            out["note"] = note
        return out


# ------------------------------------------------------------------ model
def make_layers(cfg_name: str, dev, tp_rank: int, tp_size: int, seed: int = 1234):
    """Random-init packed layers (normal x 0.02) for this rank + per-layer k."""
    import paper_2602_00397_b200 as ff
    d, f, L, T, keep = CONFIGS[cfg_name]
    ks = config_ks(cfg_name)
    r, rc = ff.default_reduced_dim(d), ff.default_comp_dim(d)
    layers = []
    g = torch.Generator(device=dev)
    for l in range(L):
        g.manual_seed(seed * 1000 + l)

        def w(*shape):
            return torch.randn(shape, generator=g, device=dev, dtype=torch.float32).mul_(0.02)

        w_gate, w_up, w_down = w(d, f), w(d, f), w(f, d)
        comp = ff.CompensatorParams(w1=w(d, rc), w2=w(rc, d))
        packed = ff.pack_layer(w_gate, w_up, w_down, comp, device=dev, tp_rank=tp_rank,
                               tp_size=tp_size)
        dp = ff.DevicePredictor(query=w(d), w1=w(d, r), w2=w(r, f))
        del w_gate, w_up, w_down
        layers.append((packed, dp, ks[l]))
    torch.cuda.synchronize(dev)
    return layers, ks


# ------------------------------------------------------------------ CPU legs
_CPU_WEIGHTS: dict = {}


def cpu_sample(cfg_name: str, impl: str, n_sparse: int = 1, seed: int = 1234):
    """Time the reference's per-block FFN branch on the host for a bounded sample.

    Returns (ms per layer extrapolated to the full block count, details).
    impl "reference": the unmodified sparseprefill package (baseline/_ref);
    impl "port": the oracle restatement (oracle/ffwd_oracle.py).
    """
    d, f, L, T, keep = CONFIGS[cfg_name]
    k = min(f, max(1, int(np.floor(keep * f + 0.5))))
    from oracle import ffwd_oracle as orc
    key = (cfg_name, 1234)
    if key not in _CPU_WEIGHTS:  # generated once; each step draws a fresh block of inputs
        rng = np.random.default_rng(1234)
        _CPU_WEIGHTS[key] = (
            {"w_gate": orc.gaussian(rng, (d, f), 0.02), "w_up": orc.gaussian(rng, (d, f), 0.02),
             "w_down": orc.gaussian(rng, (f, d), 0.02)},
            orc.init_predictor(rng, d, f), orc.init_compensator(rng, d))
    lw, pred, comp = _CPU_WEIGHTS[key]
    xb = np.random.default_rng(seed).standard_normal((128, d)).astype(np.float32)
    n_blk = -(-T // 128)
    if impl == "reference":
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        from sparseprefill.compensator import (CompensatorParams, apply_compensation,
                                               compensator_forward)
        from sparseprefill.engine import dense_ffn
        from sparseprefill.model import LayerWeights
        from sparseprefill.predictor import PredictorParams, predictor_forward
        from sparseprefill.sparse import build_mask, select_subweights, sparse_ffn_forward
        rlw = LayerWeights(wq=None, wk=None, wv=None, wo=None, w_gate=lw["w_gate"],
                           w_up=lw["w_up"], w_down=lw["w_down"], attn_norm=None, ffn_norm=None)
        rp = PredictorParams(**pred)
        rcp = CompensatorParams(**comp)

        def dense():
            return dense_ffn(xb, rlw)

        def sparse():  # engine.py:284-300
            s = predictor_forward(rp, xb)
            mask = build_mask(s, k)
            y = sparse_ffn_forward(xb, select_subweights(rlw, mask))
            return apply_compensation(y, compensator_forward(rcp, xb))
    else:
        def dense():
            return orc.dense_ffn(xb, lw["w_gate"], lw["w_up"], lw["w_down"])

        def sparse():
            s = orc.predictor_forward(pred["query"], pred["w1"], pred["w2"], xb)
            idx = orc.topk_indices(s, k)
            y = orc.sparse_ffn_forward(xb, lw["w_gate"], lw["w_up"], lw["w_down"], idx)
            return y + orc.compensator_forward(comp["w1"], comp["w2"], xb)

    t0 = time.perf_counter()
    dense()
    t_dense = time.perf_counter() - t0
    ts = []
    for _ in range(n_sparse):
        t0 = time.perf_counter()
        sparse()
        ts.append(time.perf_counter() - t0)
    t_sparse = min(ts)
    n_dense = min(2, n_blk)
    ms_layer = 1e3 * (n_dense * t_dense + (n_blk - n_dense) * t_sparse)
    return ms_layer, {"t_dense_block_s": t_dense, "t_sparse_block_s": t_sparse,
                      "n_blocks": n_blk}


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank: int, world: int) -> None:
    """The reference's own CPU implementation (baseline/_ref, unmodified) on the host cores.

    Each step is a bounded sample of the workload: one dense and one predicted 128-token
    block of one layer through the reference's per-block FFN branch (engine.py:254-310).
    `ms_per_step` is the measured wall time of that sample; `value` extrapolates it to a
    whole layer (2 dense + n-2 predicted blocks), as the `extrapolation` key states."""
    if rank != 0:
        return
    impl = "reference"
    try:
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        import sparseprefill  # noqa: F401
    except ImportError:
        impl = "port"
    d, f, L, T, keep = CONFIGS[args.config]
    if args.layers or args.tokens:
        L, T = args.layers or L, args.tokens or T
        CONFIGS[args.config] = (d, f, L, T, keep)
    layer_ms, wall_ms = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ms, info = cpu_sample(args.config, impl, n_sparse=1, seed=1234 + i)
        wall = (time.perf_counter() - t0) * 1e3
        if i >= args.warmup:
            layer_ms.append(ms)
            wall_ms.append(wall)
    v = float(np.median(layer_ms))
    n_blk = info["n_blocks"]
    n_dense = min(2, n_blk)
    sample = (f"per step: 1 dense + 1 predicted 128-token block of one layer (engine.py:254-310 "
              f"FFN branch), extrapolated to {n_dense} dense + {n_blk - n_dense} predicted blocks")
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "ms/layer",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(wall_ms)),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic (random-init normal*0.02 weights, N(0,1) hidden states)",
        "config": workload_config(args, T, L, config_ks(args.config), world),
        "extrapolation": {"measured": "1 dense + 1 predicted block per step",
                          "t_dense_block_ms": 1e3 * info["t_dense_block_s"],
                          "t_predicted_block_ms": 1e3 * info["t_sparse_block_s"],
                          "layer_ms": f"{n_dense} x t_dense + {n_blk - n_dense} x t_predicted",
                          "ms_per_step_is": "measured wall time of one step's sample"},
        "cpu_baseline": {"value": v, "unit": "ms/layer", "cores": cores(),
                         "kind": "reference" if impl == "reference" else "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "ms/layer", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ TTFT
VOCAB = 128256  # Llama-3 vocabulary (embedding + head of the TTFT model)


def measure_ttft(layers, cfg_name: str, dev, steps: int) -> dict:
    """Time-to-first-token of the full prefill (engine.prefill_blockwise semantics,
    prefill.py): embedding, 32 x (RMSNorm, QKV, RoPE, causal SDPA, Wo, RMSNorm +
    predictor logits, FFN hot path with residual), final norm and head, for the
    predicted (50%) and dense modes.  The reference architecture (model.py:18-84:
    multi-head attention, d x d Wq/Wk/Wv/Wo, head_dim 128 here) with random-init
    weights; the FFN layers are the bench's own.  Timed from host token ids to host
    last-token logits (H2D / D2H inside the region), CUDA events, mean of `steps`."""
    import paper_2602_00397_b200 as ff
    from paper_2602_00397_b200.prefill import DeviceLayer, DeviceModel, prefill
    d, f, L, T, keep = CONFIGS[cfg_name]
    cfg = ff.ModelConfig(n_layers=L, d_model=d, d_ffn=f, n_heads=d // 128, vocab_size=VOCAB,
                         max_context=T)
    g = torch.Generator(device=dev)
    g.manual_seed(4242)

    def w(*shape, dt=torch.bfloat16):
        return torch.randn(shape, generator=g, device=dev, dtype=torch.float32).mul_(0.02).to(dt)

    ones = torch.ones(d, device=dev)
    dls = [DeviceLayer(wqkv_t=w(3 * d, d), wo_t=w(d, d), attn_norm=ones, ffn_norm=ones,
                       ffn=packed, predictor=dp, k=k) for packed, dp, k in layers]
    model = DeviceModel(config=cfg, tok_emb=w(VOCAB, d, dt=torch.float32), layers=dls,
                        final_norm=ones, head=w(d, VOCAB, dt=torch.float32),
                        dense_first_last=True, attn_dtype=torch.bfloat16, has_comp=True)
    tokens = np.random.default_rng(7).integers(0, VOCAB, T)
    out = {"predicted": [], "dense": []}
    for mode in ("predicted", "dense", "predicted", "dense"):  # warm-up (cuDNN plans, pools)
        prefill(model, tokens, mode=mode).last_logits.cpu()
    torch.cuda.synchronize(dev)
    flops = {}
    for _ in range(steps):  # alternate the modes so clock / power drift hits both alike
        for mode in ("predicted", "dense"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = prefill(model, tokens, mode=mode)
            res.last_logits.cpu()
            e1.record()
            torch.cuda.synchronize(dev)
            out[mode].append(e0.elapsed_time(e1))
            flops[mode] = int(res.flops.total())
    out = {m: {"ms": statistics.mean(v), "flops": flops[m],
               "effective_tflops": flops[m] / (statistics.mean(v) * 1e-3) / 1e12}
           for m, v in out.items()}
    del model, dls
    torch.cuda.empty_cache()
    return {"unit": "ms", "T": T, "layers": L, "n_heads": cfg.n_heads, "vocab": VOCAB,
            "predicted_50pct_ms": out["predicted"]["ms"], "dense_ms": out["dense"]["ms"],
            "speedup_vs_dense": out["dense"]["ms"] / out["predicted"]["ms"],
            "predicted_effective_tflops": out["predicted"]["effective_tflops"],
            "dense_effective_tflops": out["dense"]["effective_tflops"],
            "attention": "torch SDPA (cuDNN/flash, bf16), QKV/O projections cuBLAS bf16",
            "timed": "host token ids -> host last-token logits, CUDA events, mean of "
                     f"{steps} prefills per mode (modes alternated) after 2 warm-ups each"}


# ------------------------------------------------------------------ other splits (N > 1)
def time_other_splits(args, rank: int, world: int, dev, timed, skip: str) -> dict:
    """The two splits besides the headline's, timed on the same GPUs for the extra keys:
    sequence parallel (the prompt's 128-token blocks split across ranks, weights
    replicated, no data-path collective: the FFN branch is block-local, engine.py:254-310)
    and data parallel (one independent prompt per rank, BASELINE configs[4])."""
    import paper_2602_00397_b200 as ff
    from paper_2602_00397_b200 import layer as fl
    from paper_2602_00397_b200.norm import rmsnorm
    d, f, L, T, keep = CONFIGS[args.config]
    layers, _ = make_layers(args.config, dev, 0, 1)
    n_blk = -(-T // 128)
    gain = torch.ones(d, device=dev)
    out = {}
    for mode in ("sp", "dp"):
        if mode == skip:
            continue
        gx = torch.Generator(device=dev)
        gx.manual_seed(99 + (rank if mode == "dp" else 0))
        x = torch.randn((T, d), generator=gx, device=dev).to(torch.bfloat16).float()
        dfl = True
        if mode == "sp":
            b0, b1, dfl = fl.seq_shard(n_blk, rank, world)
            x = x[b0 * 128:min(T, b1 * 128)].contiguous()
        Tl = x.shape[0]
        res = torch.empty_like(x)
        xb = torch.empty((Tl, d), dtype=torch.bfloat16, device=dev)
        lg = torch.empty((Tl,), dtype=torch.float32, device=dev)
        ws = torch.empty(max(fl.layer_workspace_bytes(Tl, p, q.r, k, dfl) for p, q, k in layers),
                         dtype=torch.uint8, device=dev)

        def st():
            res.copy_(x)
            for packed, dp, k in layers:
                rmsnorm(res, gain, out=xb, predictor=dp, logits=lg)
                ff.sparse_ffn_layer(xb, packed, dp, k, out=res, residual=res, logits_in=lg,
                                    workspace=ws, dense_first_last=dfl)

        for _ in range(max(1, args.warmup)):
            st()
        ms = timed(st, args.steps)
        prompts = world if mode == "dp" else 1
        out[mode] = {"ms_per_layer": ms / L, "prompts_per_step": prompts,
                     "prefill_ffn_tokens_per_s": prompts * T / (ms * 1e-3),
                     "scaling": "weak" if mode == "dp" else "strong",
                     "what": ("the prompt's 128-token blocks split over the ranks, weights "
                              "replicated, no collective" if mode == "sp" else
                              "one independent prompt per rank, no collective")}
        del res, xb, lg, ws
    del layers
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ GPU arm
def run_gpu(args, rank: int, world: int) -> None:
    import paper_2602_00397_b200 as ff
    from paper_2602_00397_b200 import layer as fl
    from paper_2602_00397_b200.norm import rmsnorm
    dev = torch.device("cuda", local_device())
    torch.cuda.set_device(dev)
    if args.raster:
        fl.set_raster(*(int(v) for v in args.raster.split(",")))
    peaks = load_peaks()
    d, f, L, T, keep = CONFIGS[args.config]
    if args.layers or args.tokens:
        L = args.layers or L
        T = args.tokens or T
        CONFIGS[args.config] = (d, f, L, T, keep)
    # tp: tensor parallel over d_ffn (one prompt, NCCL all-reduce per layer);
    # dp: every rank runs the whole stack on its own prompt (independent prompts, no
    # collective in the data path)
    tp = world if args.parallel == "tp" else 1
    # tp + rs_ag (the default for N > 1): sequence-parallel residual stream, all-gather of
    # the bf16 FFN input and reduce-scatter of the partial FFN output (tp.SeqParallelTP)
    rs_ag = tp > 1 and args.collective == "rs_ag"
    layers, ks = make_layers(args.config, dev, rank if tp > 1 else 0, tp)
    n_blk = -(-T // 128)
    gx = torch.Generator(device=dev)
    gx.manual_seed(99 + (rank if args.parallel == "dp" else 0))
    x0 = torch.randn((T, d), generator=gx, device=dev).to(torch.bfloat16).float()
    # sp: this rank's contiguous share of the prompt's 128-token blocks; only the ranks
    # holding the prompt's first / last block run it dense (engine.py:258-262)
    dfl, blk0, blk1 = True, 0, n_blk
    if args.parallel == "sp" and world > 1:
        blk0, blk1, dfl = fl.seq_shard(n_blk, rank, world)
        x0 = x0[blk0 * 128:min(T, blk1 * 128)].contiguous()
    gain = torch.ones(d, device=dev)            # ffn_norm gains (ones, synthetic.py:41)
    sp_tp = None
    if rs_ag:
        from paper_2602_00397_b200.tp import SeqParallelTP, TorchComm, seq_rows
        r0, r1 = seq_rows(T, rank, world)
        x0 = x0[r0:r1].contiguous()  # this rank's rows of the residual stream
        sp_tp = SeqParallelTP(layers, T, d, rank, world, dev, comm=TorchComm(), gain=gain,
                              shard_predictor={"auto": None, "sharded": True,
                                               "replicated": False}[args.predictor],
                              reduce_dtype=torch.bfloat16 if args.reduce_dtype == "bf16"
                              else torch.float32)
    T_loc = x0.shape[0]
    n_dense_loc = int(blk0 == 0) + int(blk1 == n_blk) if dfl != True else min(2, n_blk)  # noqa: E712
    n_pred_loc = (blk1 - blk0) - n_dense_loc
    res = torch.empty_like(x0)
    xb = torch.empty((T_loc, d), dtype=torch.bfloat16, device=dev)
    ybuf = torch.empty_like(x0) if tp > 1 and not rs_ag else None
    ws_bytes = max(fl.layer_workspace_bytes(T if rs_ag else T_loc, p, dp.r, k, dfl)
                   for p, dp, k in layers)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    if sp_tp is not None:
        sp_tp.workspace = ws

    lg = torch.empty((T_loc,), dtype=torch.float32, device=dev)
    peers = None
    if tp > 1 and args.collective in ("fused", "overlap"):
        # fused completion: partial Y -> peer-memory reduce + residual add (tp.PeerBuffers)
        from paper_2602_00397_b200.tp import PeerBuffers
        peers = PeerBuffers(T, d, dev, with_xnext=False)
        res = peers.out

    def stack(x_src: torch.Tensor):
        # engine.py:267-308 per layer: x = rmsnorm(h, ffn_norm) (fused with the predictor's
        # per-token logits), then predictor -> top-k -> sparse FFN + compensator, h += y
        res.copy_(x_src)
        if sp_tp is not None:  # norm on T/N rows -> AG(x, logits) -> FFN shard -> RS(y)
            sp_tp.stack(res)
            return
        for packed, dp, k in layers:
            rmsnorm(res, gain, out=xb, predictor=dp, logits=lg)
            if tp == 1:
                ff.sparse_ffn_layer(xb, packed, dp, k, out=res, residual=res, logits_in=lg,
                                    workspace=ws, dense_first_last=dfl)
            elif args.collective == "overlap":
                peers.layer_overlap(xb, packed, dp, k, residual=res, logits_in=lg,
                                    workspace=ws)
            elif peers is not None:
                ff.sparse_ffn_layer(xb, packed, dp, k, out=peers.partial, logits_in=lg,
                                    workspace=ws)
                peers.complete(res)
            else:
                ff.sparse_ffn_layer(xb, packed, dp, k, out=ybuf, logits_in=lg, workspace=ws)
                torch.distributed.all_reduce(ybuf)
                res.add_(ybuf)

    def barrier():
        if world > 1:
            if BACKEND == "nccl":
                torch.distributed.barrier(device_ids=[dev.index])
            else:
                torch.distributed.barrier()

    def timed(fn, steps):
        barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:  # max over ranks (a CPU tensor under the gloo emulation backend)
            t = torch.tensor([ms], device="cpu" if BACKEND == "gloo" else dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---- warm-up, then the timed region.  The clock sampler starts before the warm-up so
    # nvidia-smi is already sampling when the timed region begins; only rows that arrive
    # inside the timed region are kept.
    with ClockSampler(dev.index) as clk:
        for _ in range(args.warmup):
            stack(x0)
        torch.cuda.synchronize(dev)
        # the headline: uninstrumented (per-launch events would sit between the kernels and
        # defeat the programmatic-dependent-launch overlap)
        t_on = time.monotonic()
        step_ms = timed(lambda: stack(x0), args.steps)
        t_off = time.monotonic()
        time.sleep(0.35)  # let the rows sampled inside the region arrive
    if not bool(torch.isfinite(res).all()):
        raise RuntimeError("non-finite residual stream after the FFN stack")
    clocks = clk.summary(t_on, t_off)
    # the reference-exact predictor input (engine.py:267,286): the predictor pools the f32
    # RMSNorm output instead of its bf16 rounding (norm writes both; fused f32 logits)
    f32_variant = None
    if tp == 1 and not args.skip_f32_pred:
        x32 = torch.empty((T_loc, d), dtype=torch.float32, device=dev)

        def stack_f32(x_src: torch.Tensor):
            res.copy_(x_src)
            for packed, dp, k in layers:
                rmsnorm(res, gain, out=xb, out_f32=True, out32=x32, predictor=dp, logits=lg,
                        logits_from_f32=True)
                ff.sparse_ffn_layer(xb, packed, dp, k, out=res, residual=res, logits_in=lg,
                                    x_pred_f32=x32, workspace=ws, dense_first_last=dfl)

        stack_f32(x0)
        f32_ms = timed(lambda: stack_f32(x0), max(1, args.steps // 2))
        f32_variant = {"ms_per_layer": f32_ms / L, "vs_bf16_predictor_input": f32_ms / step_ms,
                       "what": "predictor pools the f32 RMSNorm output (x_pred_f32, f32 fused "
                               "logits): the reference's own predictor input; the headline's "
                               "predictor pools the bf16 FFN operand"}
        del x32
    # per-kernel breakdown and launch counts: a second, instrumented run of the same steps
    fl.timing_enable(True)
    fl.timing_read()
    timed(lambda: stack(x0), args.steps)
    fl.timing_enable(False)
    stages = fl.timing_read()

    # ---- e2e through the public API with host buffers.  Every step uploads its own input
    # from pinned host memory and reads its result back; the copies run on a copy stream,
    # double-buffered, so step i+1's upload and step i's readback overlap step i's compute
    # (the first upload and the last readback are exposed inside the timed region).
    host_in = torch.empty((T_loc, d), dtype=torch.float32, pin_memory=True)
    host_in.copy_(x0.cpu())
    host_out = [torch.empty_like(host_in, pin_memory=True) for _ in range(2)]
    xd = [torch.empty((T_loc, d), dtype=torch.float32, device=dev) for _ in range(2)]
    yd = [torch.empty((T_loc, d), dtype=torch.float32, device=dev) for _ in range(2)]
    copy_s = torch.cuda.Stream(dev)
    ev = {key: [torch.cuda.Event() for _ in range(2)] for key in ("in", "x_free", "y", "out")}

    def e2e_run(n):
        cur = torch.cuda.current_stream(dev)
        copy_s.wait_stream(cur)
        with torch.cuda.stream(copy_s):
            xd[0].copy_(host_in, non_blocking=True)
            ev["in"][0].record(copy_s)
        for i in range(n):
            j = i % 2
            if i + 1 < n:  # prefetch the next step's input into the other buffer
                with torch.cuda.stream(copy_s):
                    if i >= 1:
                        copy_s.wait_event(ev["x_free"][1 - j])
                    xd[1 - j].copy_(host_in, non_blocking=True)
                    ev["in"][1 - j].record(copy_s)
            cur.wait_event(ev["in"][j])
            stack(xd[j])
            ev["x_free"][j].record(cur)
            if i >= 2:
                cur.wait_event(ev["out"][j])  # step i-2's readback released yd[j]
            yd[j].copy_(res)
            ev["y"][j].record(cur)
            with torch.cuda.stream(copy_s):
                copy_s.wait_event(ev["y"][j])
                host_out[j].copy_(yd[j], non_blocking=True)
                ev["out"][j].record(copy_s)
        cur.wait_stream(copy_s)

    e2e_run(2)
    n_e2e = max(2, args.steps // 2)
    e2e_ms = timed(lambda: e2e_run(n_e2e), 1) / n_e2e
    torch.cuda.synchronize(dev)
    if not torch.equal(host_out[(n_e2e - 1) % 2], res.cpu()):
        raise RuntimeError("e2e readback differs from the device result")
    h2d = host_in.numel() * 4
    d2h = host_out[0].numel() * 4

    # ---- accounting
    flops_layer = [ff.ffn_path_flops(d, f, T, k) for k in ks]
    total_flops = sum(flops_layer)
    value = step_ms / L
    prompts = world if args.parallel == "dp" else 1  # prompts processed per step, all ranks
    eff_tflops = prompts * total_flops / (step_ms * 1e-3) / 1e12
    up_ms, up_n = stages["up_proj"]
    dn_ms, dn_n = stages["down_proj"]
    rc = ff.default_comp_dim(d)
    n_pred = n_pred_loc  # this rank's predicted / dense blocks (all of them unless sp)
    up_flops = sum(n_pred * (4 * 128 * d * k + 2 * 128 * d * rc) + n_dense_loc * 4 * 128 * d * f
                   for k in ks) / L
    up_avg_ms = up_ms / max(1, up_n)
    achieved = up_flops / tp / (up_avg_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(args.config, {}).get("up_proj")
    launches = sum(n for _, n in stages.values())
    w_layer = (3 * f * d + 2 * d * rc) * 2 / tp  # bf16 FFN + compensator weights, this rank

    # per-kernel rooflines: algorithmic FLOPs or bytes per launch / the
    # event-timed average launch (instrumented run), against the measured peaks
    def avg_ms(name):
        ms, n = stages.get(name, (0.0, 0))
        return ms / n if n else None

    def kroof(bound, work, ms, unit):
        if not ms:
            return None
        peak = peaks["bf16_sus"] if bound == "tensor" else peaks["hbm"]
        ach = work / (ms * 1e-3) / (1e12 if bound == "tensor" else 1e9)
        return {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                "avg_launch_ms": ms}

    r_pred = ff.default_reduced_dim(d)
    dn_flops = sum(n_pred * (2 * 128 * d * k + 2 * 128 * rc * d) + n_dense_loc * 2 * 128 * d * f
                   for k in ks) / L
    k1_bytes = sum(T_loc * d * 2 + d * r_pred * 4 + r_pred * f * 4 + 2 * n_pred * f * 4
                   + n_pred * k * 4 for k in ks) / L
    k1_ms = [avg_ms(s_) for s_ in ("pool", "predictor_w1", "predictor_w2", "topk")]
    kernels_roofline = {
        "up_proj": kroof("tensor", up_flops / tp, up_avg_ms, "TFLOP/s"),
        "down_proj": kroof("tensor", dn_flops / tp, avg_ms("down_proj"), "TFLOP/s"),
        "predictor+topk (K1: pool, W1, W2, top-k)": kroof(
            "hbm", k1_bytes, sum(m for m in k1_ms if m) if all(k1_ms) else None, "GB/s"),
        "ffn_norm (RMSNorm + predictor logits)": kroof(
            "hbm", T_loc * d * 4 + T_loc * d * 2 + T_loc * 4, avg_ms("ffn_norm"), "GB/s"),
    }

    out = {
        "metric": METRIC, "value": value, "unit": "ms/layer", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": False, "scaling": "weak" if args.parallel == "dp" and world > 1
        else "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init normal*0.02 weights, N(0,1) bf16 hidden states)",
        "config": workload_config(args, T, L, ks, world),
        "collective": ({"rs_ag": f"NCCL all-gather x (bf16) + reduce-scatter y "
                                  f"({args.reduce_dtype}), sequence-parallel residual, "
                                  + ("sequence-parallel predictor (all-gather of the "
                                     "selection bitmasks)" if sp_tp is not None and
                                     sp_tp.shard_predictor else "replicated predictor "
                                     "(all-gather of the logits)"),
                        "allreduce": "NCCL all-reduce of y (f32)", "nccl": "NCCL all-reduce "
                        "of y (f32)", "fused": "peer-memory all-reduce kernel (NVLink P2P)",
                        "overlap": "peer-memory all-reduce overlapped with the down "
                                   "projection"}[args.collective] if tp > 1 else None),
        "l2": (f"inputs larger than L2 (residual stream {T_loc * d * 4 / 2**20:.0f} MiB f32, "
               f"{w_layer / 2**20:.0f} MiB bf16 weights per layer, {L} distinct layers per "
               "step); no flush"),
        "e2e": {"value": e2e_ms / L, "unit": "ms/layer", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "api": "paper_2602_00397_b200.sparse_ffn_layer (x from pinned host f32)",
                "copies": "per step: H2D of its input, D2H of its output, on a copy stream "
                          "double-buffered against compute (first upload / last readback "
                          "exposed)", "steps": n_e2e},
        "gpu_launches": launches,
        "effective_tflops": eff_tflops,
        "prefill_ffn_tokens_per_s": prompts * T / (step_ms * 1e-3),
        "roofline": {"kernel": "up_proj (K2 gather-GEMM + SwiGLU)", "bound": "tensor",
                     "achieved": achieved, "peak": peaks["bf16_sus"], "unit": "TFLOP/s",
                     "frac": achieved / peaks["bf16_sus"],
                     "frac_of_burst": achieved / peaks["bf16"],
                     "peak_src": f"{peaks['src']} bf16 sustained (burst {peaks['bf16']})",
                     "traffic": traffic},
        "kernels_ms_per_layer": {k_: v[0] / max(1, args.steps * L) for k_, v in stages.items()},
        "kernels_roofline": kernels_roofline,
        "kernels_roofline_note": ("K1 bytes per SURVEY 8(d): X bf16 + W1 + W2 + scores + "
                                  "indices; K1 computes in f64 (exact scores), so it runs "
                                  "far below the HBM roof by design"),
        "kernels_timing": "CUDA events around each launch, in a second (instrumented) run of the same steps",
        "clocks": clocks,
        "predictor_f32_input": f32_variant,
    }

    # ---- the other splits (N > 1): extra keys on the same line
    if world > 1 and not args.skip_alt:
        del layers
        torch.cuda.empty_cache()
        out["other_splits"] = time_other_splits(args, rank, world, dev, timed, args.parallel)
        layers = None
    # ---- dense baselines on one layer (rank 0 only, single GPU)
    if world == 1 and not args.skip_dense:
        packed, dp, k = layers[0]
        xd = x0.to(torch.bfloat16)

        def own_dense_layer():  # same FFN-input norm as the sparse step, then the dense FFN
            rmsnorm(x0, gain, out=xd)
            return ff.dense_ffn(xd, packed)

        own_dense_layer()  # warm-up: workspace allocation + first-launch setup
        own_dense = timed(own_dense_layer, args.steps)
        # cuBLAS-class dense FFN: [Wg|Wu] fused GEMM, silu*mul, down GEMM (torch.matmul bf16)
        wgu = packed.wgu_t[:2 * packed.f_local]
        wdn = packed.wd[:packed.f_local]

        def cublas_ffn():
            rmsnorm(x0, gain, out=xd)
            h = xd @ wgu.t()
            a = torch.nn.functional.silu(h[:, :packed.f_local]) * h[:, packed.f_local:]
            return a @ wdn

        cublas_ffn()
        cub = timed(cublas_ffn, args.steps)
        out["dense"] = {"own_ms_per_layer": own_dense, "cublas_ms_per_layer": cub,
                        "speedup_vs_cublas_dense": cub / value,
                        "speedup_vs_own_dense": own_dense / value,
                        "dense_tflops_cublas": 6 * T * d * f / (cub * 1e-3) / 1e12}
    # ---- TTFT of the full prefill (rank 0, single GPU)
    if world == 1 and not args.skip_ttft:
        out["ttft"] = measure_ttft(layers, args.config, dev, max(1, min(4, args.steps)))
    del layers
    torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N=1): the reference's own implementation (baseline/_ref,
    # unmodified) on the host cores, else the oracle port, on a bounded sample
    if rank == 0 and world == 1 and not args.skip_cpu:
        kind = "reference"
        try:
            sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
            import sparseprefill  # noqa: F401
        except ImportError:
            kind = "port"
        ms, info = cpu_sample(args.config, kind)
        out["cpu_baseline"] = {
            "value": ms, "unit": "ms/layer", "cores": cores(), "kind": kind,
            "sample": f"{'unmodified reference package' if kind == 'reference' else 'oracle port'}"
                      f", 1 dense + 1 predicted 128-token block of one layer "
                      f"(t_dense {info['t_dense_block_s']:.2f}s, t_pred "
                      f"{info['t_sparse_block_s']:.2f}s), extrapolated to "
                      f"{info['n_blocks']} blocks"}
    if rank == 0:
        print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="8b", choices=sorted(CONFIGS))
    ap.add_argument("--layers", type=int, default=0, help="override layer count (debug)")
    ap.add_argument("--tokens", type=int, default=0, help="override prompt length (debug)")
    ap.add_argument("--skip-dense", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-ttft", action="store_true")
    ap.add_argument("--skip-f32-pred", action="store_true",
                    help="skip timing the f32-predictor-input variant")
    ap.add_argument("--predictor", default="auto", choices=["auto", "sharded", "replicated"],
                    help="TP with rs_ag: each rank predicts only its own blocks and the "
                         "selection bitmasks are all-gathered (sharded; auto = from 4 ranks), "
                         "or every rank predicts every block (replicated)")
    ap.add_argument("--collective", default="rs_ag",
                    choices=["rs_ag", "allreduce", "nccl", "fused", "overlap"],
                    help="TP completion: rs_ag = sequence-parallel residual (NCCL all-gather "
                         "of x, reduce-scatter of y; the default), allreduce (= nccl) = NCCL "
                         "all-reduce of y, fused = the peer-memory all-reduce kernel, overlap "
                         "= that kernel draining blocks while the down projection runs")
    ap.add_argument("--reduce-dtype", default="f32", choices=["f32", "bf16"],
                    help="rs_ag: dtype of the partial y reduce-scatter")
    ap.add_argument("--parallel", default="tp", choices=["tp", "sp", "dp"],
                    help="N>1: tensor parallel over d_ffn (the north star's split; default), "
                         "sequence parallel (the prompt's 128-token blocks split across GPUs, "
                         "weights replicated, no collective), or data parallel (one prompt "
                         "per GPU)")
    ap.add_argument("--skip-alt", action="store_true",
                    help="N>1: skip timing the other two splits (sp, dp) for the extra keys")
    ap.add_argument("--raster", default="", help="UP,DOWN blocks per L2 raster group (tuning)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        torch.cuda.set_device(local_device())
        if BACKEND == "nccl":  # bind the rank's GPU (barriers and collectives use it)
            # communicator lines (rank / nRanks / transports) for the run's record
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.distributed.init_process_group(
                "nccl", device_id=torch.device("cuda", local_device()))
        else:
            torch.distributed.init_process_group(BACKEND)
    try:
        run_gpu(args, rank, world)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
