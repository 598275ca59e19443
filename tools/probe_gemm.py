"""Where the gather-GEMMs' MMA thread waits (FFWD_PROBE build: tools/build_variant.sh probe
-DFFWD_PROBE; run with FFWD_LIB=build/libffwd_probe.so).  One 8B/16K layer of the bench
step, then per-CTA cycle counts of the last K2 and K3 launches.  usage: probe_gemm.py [CFG] [T]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2602_00397_b200 as ff
from paper_2602_00397_b200 import _lib
from paper_2602_00397_b200 import layer as fl
from paper_2602_00397_b200.norm import rmsnorm

cfg = sys.argv[1] if len(sys.argv) > 1 else "8b"
d, f, _, T, keep = bench.CONFIGS[cfg]
if len(sys.argv) > 2:  # token-count override (K3 with H L2-resident at small T)
    T = int(sys.argv[2])
bench.CONFIGS[cfg] = (d, f, 1, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers(cfg, dev, 0, 1)
packed, dp, k = layers[0]
gain = torch.ones(d, device=dev)
x0 = torch.randn((T, d), device=dev).to(torch.bfloat16).float()
res = torch.empty_like(x0)
xb = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
lg = torch.empty((T,), dtype=torch.float32, device=dev)
ws = torch.empty(fl.layer_workspace_bytes(T, packed, dp.r, k, True), dtype=torch.uint8, device=dev)
lib = _lib.load_library()
for it in range(3):
    res.copy_(x0)
    rmsnorm(res, gain, out=xb, predictor=dp, logits=lg)
    ff.sparse_ffn_layer(xb, packed, dp, k, out=res, residual=res, logits_in=lg, workspace=ws)
torch.cuda.synchronize()
for tag in ("up", "down"):
    buf = (ctypes.c_ulonglong * (256 * 5))()
    getattr(lib, f"ffwd_probe_read_{tag}")(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(256, 5)[:148].astype(np.float64)
    tot = a[:, 3]
    print(f"T={T} {tag}: total {tot.mean():.0f} cyc/CTA; MMA thread waiting on A {a[:, 0].sum() / tot.sum() * 100:.1f}%, "
          f"on B {a[:, 1].sum() / tot.sum() * 100:.1f}%, on the epilogue (TMEM) {a[:, 2].sum() / tot.sum() * 100:.1f}%; "
          f"stages/CTA {a[:, 4].mean():.0f}, cycles/stage {tot.sum() / a[:, 4].sum():.0f}; "
          f"CTA total min/max {tot.min():.0f}/{tot.max():.0f}")
