"""A/B of the TTFT model (bench.measure_ttft) with a few layers: fused vs unfused logits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2602_00397_b200.prefill as pf

cfg = sys.argv[1] if len(sys.argv) > 1 else "8b"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
d, f, _, T, keep = bench.CONFIGS[cfg]
bench.CONFIGS[cfg] = (d, f, L, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers(cfg, dev, 0, 1)
for fuse in (True, False, True, False):
    pf.FUSE_LOGITS = fuse
    r = bench.measure_ttft(layers, cfg, dev, 3)
    print(f"fuse={fuse}: predicted {r['predicted_50pct_ms'] / L:.3f} ms/layer, "
          f"dense {r['dense_ms'] / L:.3f} ms/layer")
