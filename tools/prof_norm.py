"""FFN-input RMSNorm (+ fused predictor logits) at the 8B/16K shape: ncu target + timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_00397_b200 as ff
from paper_2602_00397_b200.norm import rmsnorm

T, d, f, r = 16384, 4096, 14336, 256
dev = torch.device("cuda", 0)
x = torch.randn((T, d), device=dev)
gain = torch.ones(d, device=dev)
dp = ff.DevicePredictor(query=torch.randn(d, device=dev) * 0.02, w1=torch.zeros((d, r), device=dev),
                        w2=torch.zeros((r, f), device=dev))
xb = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
lg = torch.empty(T, device=dev)
for _ in range(3):
    rmsnorm(x, gain, out=xb, predictor=dp, logits=lg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ("with logits", "norm only"):
    e0.record()
    for _ in range(20):
        rmsnorm(x, gain, out=xb, predictor=dp if mode == "with logits" else None, logits=lg)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{mode}: {ms * 1e3:.1f} us, {(T * d * 6) / (ms * 1e-3) / 1e9:.0f} GB/s")
