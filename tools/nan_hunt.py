"""Locate non-finite values in the 8B FFN stack, layer by layer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2602_00397_b200 as ff
from paper_2602_00397_b200 import layer as fl

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
d, f, _, T, keep = bench.CONFIGS["8b"]
bench.CONFIGS["8b"] = (d, f, L, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers("8b", dev, 0, 1)
x0 = torch.randn((T, d), device=dev).to(torch.bfloat16).float()
res = x0.clone()
xb = x0.to(torch.bfloat16)
ws = torch.empty(max(fl.layer_workspace_bytes(T, p, dp.r, k, True) for p, dp, k in layers),
                 dtype=torch.uint8, device=dev)
for l, (p, dp, k) in enumerate(layers):
    xin = xb.clone()
    y, idx = ff.sparse_ffn_layer(xb, p, dp, k, return_indices=True, workspace=ws)
    bad = ~torch.isfinite(y)
    rows = bad.any(1).nonzero().flatten()
    print(f"layer {l}: |x| rms {xin.float().pow(2).mean().sqrt():.3f}, y rms "
          f"{y[torch.isfinite(y)].pow(2).mean().sqrt():.3f}, non-finite {int(bad.sum())} in "
          f"{rows.numel()} rows, blocks {sorted(set((rows // 128).tolist()))[:10]}, "
          f"idx min/max {int(idx.min())}/{int(idx.max())}, idx sorted "
          f"{bool((idx[:, 1:] > idx[:, :-1]).all())}", flush=True)
    if rows.numel():
        r = int(rows[0])
        print("   first bad row", r, "x finite:", bool(torch.isfinite(xin[r].float()).all()),
              "cols", bad[r].nonzero().flatten()[:8].tolist())
        # dense reference for that block via torch
        b = r // 128
        xr = xin[b * 128:(b + 1) * 128].float()
        g = xr @ p.wgu_t[:f].float().t()
        u = xr @ p.wgu_t[f:2 * f].float().t()
        print("   gate max", float(g.abs().max()), "up max", float(u.abs().max()))
        break
    res = res + y
    xb = res.to(torch.bfloat16)
