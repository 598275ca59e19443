"""Single-GPU proxy of one tensor-parallel rank's compute per layer (no collectives):
the 8B shape at T=16384 split over N ranks, rank 0's strided d_ffn shard.

  replicated  the FFN shard over all T tokens with the predictor and top-k over every
              block (each rank recomputes the global selection)
  sharded     predict_mask of the rank's own T/N / 128 blocks + the FFN shard over all T
              tokens from the (gathered) bitmasks
(the FFN-input norm on the rank's T/N rows is the same in both and left out)

usage: tp_rank_proxy.py [N ...]   -> one line per N: ms/layer of both, and the K1 share."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_00397_b200 as ff  # noqa: E402

d, f, _, T, keep = bench.CONFIGS["8b"]
dev = torch.device("cuda", 0)
L = 4


def timed(fn, steps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps / L


for N in [int(v) for v in sys.argv[1:]] or [1, 2, 4, 8]:
    bench.CONFIGS["8b"] = (d, f, L, T, keep)
    layers, ks = bench.make_layers("8b", dev, 0, N)
    n = T // N
    x_full = torch.randn((T, d), device=dev).to(torch.bfloat16)
    lg_full = torch.randn((T,), device=dev) * 0.01
    y = torch.empty((T, d), dtype=torch.float32, device=dev)
    n_blk = T // 128
    mask = torch.zeros((n_blk, ff.mask_words(f)), dtype=torch.int32, device=dev)
    ws = torch.empty(max(ff.layer.layer_workspace_bytes(T, p, q.r, k, True) for p, q, k in layers),
                     dtype=torch.uint8, device=dev)
    nbr = n_blk // N

    def replicated():
        for packed, dp, k in layers:
            ff.sparse_ffn_layer(x_full, packed, dp, k, out=y, logits_in=lg_full, workspace=ws)

    # the other ranks' bitmasks (gathered in a real run): each layer's selection of
    # every block, so both variants run the same neurons
    masks = []
    for packed, dp, k in layers:
        m = torch.zeros_like(mask)
        ff.predict_mask(x_full, dp, k, blk_begin=1, blk_count=n_blk - 2, logits_in=lg_full,
                        out=m[1:n_blk - 1])
        masks.append(m)
    xr, lr = x_full[:n], lg_full[:n]  # rank 0's rows (the norm's output in a real run)

    def sharded():
        for (packed, dp, k), m in zip(layers, masks):
            # rank 0's own blocks but the dense first (and, alone, the dense last)
            ff.predict_mask(xr, dp, k, blk_begin=1, blk_count=nbr - 1 - (N == 1), logits_in=lr,
                            out=m[1:nbr - (N == 1)])
            ff.sparse_ffn_layer(x_full, packed, dp, k, out=y, mask_in=m, workspace=ws)
    ra, rb = [], []
    for _ in range(3):  # alternate, keep the best of each (boxes drift under the power cap)
        ra.append(timed(replicated))
        rb.append(timed(sharded))
    a, b = min(ra), min(rb)
    print(f"TP={N}: per-rank ms/layer replicated {a:.4f} sharded {b:.4f} "
          f"(saves {a - b:.4f} ms, {100 * (a - b) / a:.1f}%)", flush=True)
    del layers
    torch.cuda.empty_cache()
