"""TP completion on one GPU (tp_size 1, so the 'peers' are this GPU): how much of the
completion the overlapped path hides behind the down projection.

  local    sparse_ffn_layer with the residual add fused into K3 (no completion at all)
  seq      layer -> partial Y, then ffwd_allreduce_residual (reads partial + residual,
           writes the output: 768 MB per 8B/16K layer)
  overlap  ffwd_ffn_layer_tp_overlap: the same completion drained block by block while
           K3 still runs (comm_ctas CTAs beside K3's)

usage: python tools/overlap_ab.py [cfg] [layers] [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2602_00397_b200 as ff
from paper_2602_00397_b200.layer import layer_workspace_bytes
from paper_2602_00397_b200.tp import allreduce_residual_fused, sparse_ffn_layer_tp_overlap

cfg = sys.argv[1] if len(sys.argv) > 1 else "8b"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
d, f, _, T, keep = bench.CONFIGS[cfg]
bench.CONFIGS[cfg] = (d, f, L, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers(cfg, dev, 0, 1)
xb = torch.randn((T, d), device=dev).to(torch.bfloat16)
res = torch.randn((T, d), device=dev)
part = torch.empty_like(res)
ws = torch.empty(max(layer_workspace_bytes(T, p, dp.r, k, True) for p, dp, k in layers),
                 dtype=torch.uint8, device=dev)
flags = torch.zeros(3, dtype=torch.int32, device=dev)
y_done = torch.zeros(-(-T // 128), dtype=torch.int32, device=dev)
comm = torch.cuda.Stream(dev)
state = {"epoch": 0, "y_epoch": 0}


def run(mode):
    for packed, dp, k in layers:
        if mode == "local":
            ff.sparse_ffn_layer(xb, packed, dp, k, out=res, residual=res, workspace=ws)
        elif mode == "seq":
            ff.sparse_ffn_layer(xb, packed, dp, k, out=part, workspace=ws)
            state["epoch"] += 1
            allreduce_residual_fused([part], [res], [flags], 0, res, state["epoch"])
        else:
            state["epoch"] += 1
            state["y_epoch"] += 1
            sparse_ffn_layer_tp_overlap(
                xb, packed, dp, k, partials=[part], outs=[res], flags=[flags], y_done=[y_done],
                residual=res, epoch=state["epoch"], y_epoch=state["y_epoch"],
                comm_ctas=int(mode.split(":")[1]), workspace=ws, comm_stream=comm)


def timed(mode):
    run(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        run(mode)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (iters * L)


modes = ["local", "seq", "overlap:8", "overlap:16", "overlap:32"]
out = {m: [] for m in modes}
for _ in range(3):
    for m in modes:
        out[m].append(timed(m))
for m in modes:
    print(f"{cfg} T={T} {m:11s} ms/layer " + " ".join(f"{v:.3f}" for v in out[m]))
