"""One 8B-shape layer, a few iterations: target for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2602_00397_b200 as ff

cfg = sys.argv[1] if len(sys.argv) > 1 else "8b"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = sys.argv[3] if len(sys.argv) > 3 else "sparse"
if len(sys.argv) > 4:  # raster groups "UP,DOWN"
    ff.set_raster(*(int(v) for v in sys.argv[4].split(",")))
if len(sys.argv) > 5:  # serpentine 0/1
    from paper_2602_00397_b200 import _lib
    _lib.load_library().ffwd_set_serpentine(int(sys.argv[5]))
d, f, L, T, keep = bench.CONFIGS[cfg]
if os.environ.get("FFWD_T"):  # token-count override
    T = int(os.environ["FFWD_T"])
bench.CONFIGS[cfg] = (d, f, 1, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers(cfg, dev, 0, 1)
packed, dp, k = layers[0]
x = torch.randn((T, d), device=dev).to(torch.bfloat16)
for _ in range(iters):
    if mode == "dense":
        ff.dense_ffn(x, packed)
    else:
        ff.sparse_ffn_layer(x, packed, dp, k)
torch.cuda.synchronize()
print("done")
