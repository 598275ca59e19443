"""Sequence parallelism over the prompt's 128-token blocks (bench.py --parallel sp): the
FFN branch is block-local (engine.py:254-310), so shards of the prompt run independently
with replicated weights.  Bar: the shards' outputs and selected indices equal the
whole-prompt call bit for bit (serpentine K order off: it reverses the accumulation order
of odd raster groups, which depend on the shard), and within 1e-6 with it on."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ff():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_00397_b200 as ff
    from paper_2602_00397_b200 import _lib
    _lib.require_device(torch.cuda.current_device())
    return ff


def _layer(ff, d=512, f=1376, seed=3):
    g = torch.Generator(device="cuda").manual_seed(seed)

    def w(*shape):
        return torch.randn(shape, generator=g, device="cuda").mul_(0.02)

    comp = ff.CompensatorParams(w1=w(d, 64), w2=w(64, d))
    packed = ff.pack_layer(w(d, f), w(d, f), w(f, d), comp, device="cuda")
    dp = ff.DevicePredictor(query=w(d), w1=w(d, 32), w2=w(32, f))
    return packed, dp


@pytest.mark.parametrize("shards,T", [(2, 1024), (4, 2048), (3, 1280)])
def test_sequence_shards_match_whole_prompt(ff, shards, T):
    from paper_2602_00397_b200 import _lib
    lib = _lib.load_library()
    packed, dp = _layer(ff)
    d = packed.d
    k = ff.budget_to_k(0.5, packed.f_global)
    x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    n_blk = T // 128
    for serp in (0, 1):
        lib.ffwd_set_serpentine(serp)
        try:
            y_all, idx_all = ff.sparse_ffn_layer(x, packed, dp, k, return_indices=True)
            parts, idxs = [], []
            for r in range(shards):
                b0, b1 = n_blk * r // shards, n_blk * (r + 1) // shards
                dfl = "first" if r == 0 else ("last" if r == shards - 1 else False)
                y, idx = ff.sparse_ffn_layer(x[b0 * 128:b1 * 128], packed, dp, k,
                                             dense_first_last=dfl, return_indices=True)
                parts.append(y)
                idxs.append(idx)
            y_sp, idx_sp = torch.cat(parts), torch.cat(idxs)
        finally:
            lib.ffwd_set_serpentine(1)
        assert torch.equal(idx_sp, idx_all), "selected neurons differ between shards and whole"
        if serp == 0:
            assert torch.equal(y_sp, y_all)
        else:
            rel = float((y_sp - y_all).norm() / y_all.norm())
            assert rel < 1e-6, rel


def test_dense_first_last_codes(ff):
    """'first' / 'last' keep exactly one dense block; bad values are rejected."""
    packed, dp = _layer(ff)
    k = ff.budget_to_k(0.5, packed.f_global)
    x = torch.randn((512, packed.d), device="cuda").to(torch.bfloat16)
    for dfl, n_pred in ((True, 2), ("first", 3), ("last", 3), (False, 4)):
        _, idx = ff.sparse_ffn_layer(x, packed, dp, k, dense_first_last=dfl,
                                     return_indices=True)
        assert idx.shape[0] == n_pred
    with pytest.raises(ff.ValidationError):
        ff.sparse_ffn_layer(x, packed, dp, k, dense_first_last="middle")


@pytest.mark.parametrize("parallel", [None, "sharded", "sp", "dp"])
def test_bench_multi_rank_runs(ff, parallel):
    """bench.py under torchrun, 2 ranks, emulated on the one GPU (gloo rendezvous, both
    ranks time-sliced on GPU 0). Default (None) = tensor parallel over d_ffn (the north
    star's split) with the sequence-parallel residual; sp = the prompt's blocks split with
    no collective; dp = one prompt per rank (BASELINE configs[4], weak scaling); sharded =
    the default split with the sequence-parallel predictor (each rank predicts its own
    blocks, the selection bitmasks are all-gathered). The JSON line must be well formed
    and name the split."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, FFWD_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2",
           "--config", "1b", "--layers", "2", "--steps", "2", "--warmup", "3"]
    if parallel == "sharded":
        cmd += ["--predictor", "sharded"]
    elif parallel is not None:
        cmd += ["--parallel", parallel]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=400)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    want = {None: "tp2", "sharded": "tp2", "sp": "sp2", "dp": "dp2"}[parallel]
    if parallel == "sharded":
        assert "sequence-parallel predictor" in d["collective"]
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == want
    assert d["scaling"] == ("weak" if parallel == "dp" else "strong")
    assert d["value"] > 0 and d["e2e"]["value"] > 0
