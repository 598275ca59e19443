"""Adjacent-block selection overlap at 8B/16K (bench weights, random inputs): the union size a block-pair K3 would gather."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2602_00397_b200 as ff
d, f, _, T, keep = bench.CONFIGS["8b"]
bench.CONFIGS["8b"] = (d, f, 1, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers("8b", dev, 0, 1)
packed, dp, k = layers[0]
x = torch.randn((T, d), device=dev).to(torch.bfloat16)
_, idx = ff.sparse_ffn_layer(x, packed, dp, k, return_indices=True)
m = torch.zeros((idx.shape[0], f), dtype=torch.bool, device=dev)
m.scatter_(1, idx.long(), True)
u = (m[0::2] | m[1::2]).sum(1).float() / f
inter = (m[0::2] & m[1::2]).sum(1).float() / k
print(f"adjacent-pair union / d_ffn: mean {u.mean():.3f} (min {u.min():.3f}, max {u.max():.3f}); overlap / k: {inter.mean():.3f}")
