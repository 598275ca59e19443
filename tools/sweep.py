"""Sparsity x length sweep on the Llama-3.1-8B FFN shape (BASELINE configs[4], 1 GPU).

keep in {75, 50, 25}% (sparsity 25/50/75%) x T in {1K, 4K, 8K, 16K, 28K}: ms/layer of the
FFN branch (FFN-input RMSNorm fused with the predictor logits, predictor + top-k +
gather-GEMMs + compensator + fused residual, dense first/last block) over a 4-layer
stack with distinct weights, against this build's dense FFN and the cuBLAS-class dense
FFN (torch.matmul bf16: fused gate/up GEMM, SiLU*up, down GEMM), each behind the same
RMSNorm, on the same layer.  One JSON line per point on stdout.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_00397_b200 as ff  # noqa: E402
from paper_2602_00397_b200 import layer as fl  # noqa: E402
from paper_2602_00397_b200.norm import rmsnorm  # noqa: E402

L = 4
KEEPS = (0.75, 0.5, 0.25)
TS = (1024, 4096, 8192, 16384, 28672)
STEPS = 5


def timed(fn, steps=STEPS):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    dev = torch.device("cuda", 0)
    d, f, _, _, _ = bench.CONFIGS["8b"]
    bench.CONFIGS["8b"] = (d, f, L, 16384, 0.5)
    layers, _ = bench.make_layers("8b", dev, 0, 1)
    gain = torch.ones(d, device=dev)
    for T in TS:
        x0 = torch.randn((T, d), device=dev).to(torch.bfloat16).float()
        xb = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
        lg = torch.empty((T,), dtype=torch.float32, device=dev)
        packed = layers[0][0]
        wgu, wdn = packed.wgu_t[:2 * f], packed.wd[:f]

        def cublas_ffn():
            rmsnorm(x0, gain, out=xb)
            h = xb @ wgu.t()
            a = torch.nn.functional.silu(h[:, :f]) * h[:, f:]
            return a @ wdn

        def own_dense():
            rmsnorm(x0, gain, out=xb)
            return ff.dense_ffn(xb, packed)

        cub = timed(cublas_ffn)
        own = timed(own_dense)
        res = torch.empty((T, d), dtype=torch.float32, device=dev)
        for keep in KEEPS:
            k = ff.budget_to_k(keep, f)
            ws = torch.empty(max(fl.layer_workspace_bytes(T, p, dp.r, k, True)
                                 for p, dp, _ in layers), dtype=torch.uint8, device=dev)

            def stack():
                res.copy_(x0)
                for p, dp, _ in layers:
                    rmsnorm(res, gain, out=xb, predictor=dp, logits=lg)
                    ff.sparse_ffn_layer(xb, p, dp, k, out=res, residual=res, logits_in=lg,
                                        workspace=ws)

            ms = timed(stack) / L
            flops = ff.ffn_path_flops(d, f, T, k)
            print(json.dumps({
                "config": "Llama-3.1-8B FFN shape", "T": T, "sparsity": round(1 - keep, 2),
                "keep": keep, "k": k, "ms_per_layer": ms, "dense_own_ms": own,
                "dense_cublas_ms": cub, "speedup_vs_cublas": cub / ms,
                "speedup_vs_own_dense": own / ms, "effective_tflops": flops / (ms * 1e-3) / 1e12,
                "layers_timed": L, "steps": STEPS}), flush=True)
            del ws
        assert torch.isfinite(res).all(), "non-finite residual stream"
        del x0, res, xb
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
