"""CTA-pair down projection (down_pair.cu) against the single-block K3, 8B shape, T=16K:
correctness of the pair kernel on synthetic H (pair i = blocks 2i, 2i+1 sharing index row
2i's first 64 nk neurons) and its time against down_proj over the same MMA work.
Build: tools/build_variant.sh pair -DFFWD_PAIR_BENCH; run with FFWD_LIB=build/libffwd_pair.so."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_00397_b200 as ff  # noqa: E402
from paper_2602_00397_b200 import _dev, _lib  # noqa: E402
from paper_2602_00397_b200 import layer as fl  # noqa: E402

d, f, _, T, keep = bench.CONFIGS["8b"]
bench.CONFIGS["8b"] = (d, f, 1, T, keep)
dev = torch.device("cuda", 0)
layers, ks = bench.make_layers("8b", dev, 0, 1)
packed, dp, k = layers[0]
lib = _lib.load_library()
fn = lib.ffwd_down_pair_bench
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
               ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
               ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
x = torch.randn((T, d), device=dev).to(torch.bfloat16)
_, idx = ff.sparse_ffn_layer(x, packed, dp, k, return_indices=True)
n_blk = T // 128
n_pairs = n_blk // 2 - 1            # pairs over blocks 0 .. 2 n_pairs - 1 (idx rows)
nk = k // 64
hcols = nk * 64
H = (torch.randn((n_blk * 128, hcols), device=dev) * 0.05).to(torch.bfloat16)
y = torch.zeros((T, d), device=dev)
stream = _dev.stream_handle(dev)
idx = idx.contiguous()
rc = fn(H.data_ptr(), hcols, packed.wd.data_ptr(), packed.wd.shape[0], T, d, y.data_ptr(), None,
        idx.data_ptr(), idx.shape[1], n_pairs, nk, stream)
torch.cuda.synchronize()
assert rc == 0, rc
wd = packed.wd.float()
worst = 0.0
for i in (0, n_pairs // 2, n_pairs - 1):
    rows = idx[2 * i, :hcols].long()
    for b in (2 * i, 2 * i + 1):
        ref = H[b * 128:(b + 1) * 128].float() @ wd[rows]
        got = y[b * 128:(b + 1) * 128]
        rel = float((got - ref).norm() / ref.norm())
        worst = max(worst, rel)
print(f"pair kernel rel-L2 vs torch (f32 of the same bf16 operands): worst {worst:.2e}")


def timed(run, steps=10):
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


t_pair = timed(lambda: fn(H.data_ptr(), hcols, packed.wd.data_ptr(), packed.wd.shape[0], T, d,
                          y.data_ptr(), None, idx.data_ptr(), idx.shape[1], n_pairs, nk, stream))
# single-block K3 over the same blocks and lists (2 n_pairs blocks, the first hcols
# entries of each row): run_sparse_ffn with per-block indices, K3 time from the timing hook
xs = x[:2 * n_pairs * 128].contiguous()
idx_s = idx[:2 * n_pairs, :hcols].contiguous()
fl.timing_enable(True)
fl.timing_read()
for _ in range(10):
    ff.run_sparse_ffn(xs, packed, idx_s, hcols)
torch.cuda.synchronize()
t = fl.timing_read()
fl.timing_enable(False)
t_down = t["down_proj"][0] / t["down_proj"][1]
stages = 2 * n_pairs * (d // 256) * nk
print(f"pair kernel {t_pair:.3f} ms  vs  down_proj {t_down:.3f} ms over the same "
      f"{stages} block-stages ({2 * n_pairs} blocks x {d // 256} column tiles x {nk} stages)")
