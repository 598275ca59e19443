"""What holds the down projection (K3) back: gathers themselves or their L2 misses?

run_sparse_ffn (K2 + K3, no predictor) at 8B/16K, k = 7168, with three index patterns:
  perblock  every 128-token block its own sorted random neuron subset (the real case)
  shared    one sorted random subset for all blocks (same gathers, W_down rows L2-hot)
  dense     identity over all neurons (2-D tile loads, no gathers; 2x the work)
Run under ncu (-k regex:down_proj) for per-kernel tensor-pipe / L2 numbers.

usage: python tools/k3_locality.py [pattern ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2602_00397_b200 as ff
from paper_2602_00397_b200.layer import run_sparse_ffn

d, f, _, T, keep = bench.CONFIGS["8b"]
bench.CONFIGS["8b"] = (d, f, 1, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers("8b", dev, 0, 1)
packed, _, k = layers[0]
x = torch.randn((T, d), device=dev).to(torch.bfloat16)
n_blk = T // 128
g = torch.Generator(device=dev).manual_seed(5)


def subset():
    return torch.sort(torch.randperm(f, generator=g, device=dev)[:k])[0].to(torch.int32)


pats = sys.argv[1:] or ["perblock", "shared", "dense"]
for pat in pats:
    if pat == "perblock":
        idx = torch.stack([subset() for _ in range(n_blk)])
        run = lambda: run_sparse_ffn(x, packed, idx, k)  # noqa: E731
    elif pat == "shared":
        idx = subset().reshape(1, k)
        run = lambda: run_sparse_ffn(x, packed, idx, k, idx_per_block=False)  # noqa: E731
    else:
        run = lambda: ff.dense_ffn(x, packed)  # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    print(f"{pat:9s} {e0.elapsed_time(e1) / 5:.3f} ms (K2+K3+plan)")
