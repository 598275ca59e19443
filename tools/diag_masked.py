import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2602_00397_b200 as ff
from paper_2602_00397_b200 import layer as fl
d, f, _, T, keep = bench.CONFIGS["8b"]
bench.CONFIGS["8b"] = (d, f, 2, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers("8b", dev, 0, 1)
x = torch.randn((T, d), device=dev).to(torch.bfloat16)
lg = torch.randn((T,), device=dev) * 0.01
y = torch.empty((T, d), dtype=torch.float32, device=dev)
n_blk = T // 128
ws = torch.empty(fl.layer_workspace_bytes(T, layers[0][0], layers[0][1].r, layers[0][2], True), dtype=torch.uint8, device=dev)
masks = []
for p, dp, k in layers:
    m = torch.zeros((n_blk, ff.mask_words(f)), dtype=torch.int32, device=dev)
    ff.predict_mask(x, dp, k, blk_begin=1, blk_count=n_blk - 2, logits_in=lg, out=m[1:n_blk-1]); masks.append(m)
def run(mode):
    for (p, dp, k), m in zip(layers, masks):
        if mode == "rep": ff.sparse_ffn_layer(x, p, dp, k, out=y, logits_in=lg, workspace=ws)
        elif mode == "mask": ff.sparse_ffn_layer(x, p, dp, k, out=y, mask_in=m, workspace=ws)
        else: ff.predict_mask(x, dp, k, blk_begin=1, blk_count=n_blk - 2, logits_in=lg, out=m[1:n_blk-1])
for mode in ("rep", "mask", "pred", "rep", "mask", "pred"):
    run(mode); torch.cuda.synchronize()
    fl.timing_enable(True); fl.timing_read()
    for _ in range(3): run(mode)
    torch.cuda.synchronize()
    t = fl.timing_read(); fl.timing_enable(False)
    print(mode, {k: round(v[0] / 6, 4) for k, v in t.items() if v[1]})


def timed(fn, steps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps / len(layers)


def both():
    run("pred")
    run("mask")


for _ in range(3):
    print("whole-layer ms: replicated %.4f  predict_mask + masked %.4f" % (timed(lambda: run("rep")), timed(both)))
