"""The bench's per-layer step (FFN-input RMSNorm + fused logits -> sparse_ffn_layer with the
fused residual) on a small stack of one BASELINE config: ncu target for every kernel of
the step.  usage: prof_step.py [CFG] [LAYERS] [ITERS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2602_00397_b200 as ff
from paper_2602_00397_b200 import layer as fl
from paper_2602_00397_b200.norm import rmsnorm

cfg = sys.argv[1] if len(sys.argv) > 1 else "8b"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
d, f, _, T, keep = bench.CONFIGS[cfg]
bench.CONFIGS[cfg] = (d, f, L, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers(cfg, dev, 0, 1)
gain = torch.ones(d, device=dev)
x0 = torch.randn((T, d), device=dev).to(torch.bfloat16).float()
res = torch.empty_like(x0)
xb = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
lg = torch.empty((T,), dtype=torch.float32, device=dev)
ws = torch.empty(max(fl.layer_workspace_bytes(T, p, q.r, k, True) for p, q, k in layers),
                 dtype=torch.uint8, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(iters):
    res.copy_(x0)
    e0.record()
    for packed, dp, k in layers:
        rmsnorm(res, gain, out=xb, predictor=dp, logits=lg)
        ff.sparse_ffn_layer(xb, packed, dp, k, out=res, residual=res, logits_in=lg, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"iter {it}: {e0.elapsed_time(e1) / L:.3f} ms/layer")
assert torch.isfinite(res).all()
print("done")
