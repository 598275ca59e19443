"""Full prefill (TTFT model of bench.py) with a few layers: target for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_00397_b200.prefill import prefill

cfg = sys.argv[1] if len(sys.argv) > 1 else "8b"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = sys.argv[3] if len(sys.argv) > 3 else "predicted"
d, f, _, T, keep = bench.CONFIGS[cfg]
bench.CONFIGS[cfg] = (d, f, L, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers(cfg, dev, 0, 1)
r = bench.measure_ttft(layers, cfg, dev, 1)
print(r)
