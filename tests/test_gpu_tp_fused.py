"""Fused tensor-parallel completion (peer-memory reduce-scatter + all-gather with the
residual add fused in, ``ffwd_allreduce_residual``), emulated on one GPU: every
"rank" has its own partial / output / flag buffers on the device and its own stream,
so the cross-rank flag protocol runs for real (the ranks' kernels are co-resident and
wait on each other); only the NVLink hop is missing.  Bar: bit-exact against
residual + sum of partials in rank order; the layer-level test checks the TP shards'
completion against the unsharded layer within the FFN tolerance."""

import numpy as np
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


def _run_ranks(partials, outs, flags, residuals, epoch, xnexts=None):
    from paper_2602_00397_b200.tp import allreduce_residual_fused
    n = len(partials)
    streams = [torch.cuda.Stream() for _ in range(n)]
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for r in range(n):
        with torch.cuda.stream(streams[r]):
            allreduce_residual_fused(partials, outs, flags, r, residuals[r], epoch, xnexts,
                                     max_ctas=max(1, 120 // n))
    for s in streams:
        cur.wait_stream(s)
    torch.cuda.synchronize()


@pytest.mark.parametrize("n,T,d", [(2, 300, 256), (4, 1000, 512), (8, 129, 64)])
def test_fused_completion_bit_exact(ff, n, T, d):
    g = torch.Generator(device="cuda").manual_seed(n)
    partials = [torch.randn((T, d), generator=g, device="cuda") for _ in range(n)]
    residual = torch.randn((T, d), generator=g, device="cuda")
    want = residual.clone()
    for p in partials:
        want = want + p  # fixed rank order, like the kernel
    flags = [torch.zeros(2 * n + 1, dtype=torch.int32, device="cuda") for _ in range(n)]
    for epoch in (1, 2):  # flags are reused across calls with increasing epochs
        # residual aliases each rank's output (the residual stream updated in place)
        outs = [residual.clone() for _ in range(n)]
        xn = [torch.empty((T, d), dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        _run_ranks(partials, outs, flags, outs, epoch, xn)
        for r in range(n):
            assert torch.equal(outs[r], want), f"rank {r} output differs (epoch {epoch})"
            assert torch.equal(xn[r], want.to(torch.bfloat16))
    for f in flags:
        assert int(f[2 * n]) == 0  # grid counter re-armed


def test_fused_completion_of_sharded_layer(ff):
    """TP=2 and 4 shards of one 8B-shaped layer slice (d 512, f 1376, T 512): partials
    from the sharded sparse FFN, completed by the fused kernel, equal the unsharded
    layer's fused-residual output within the FFN tolerance, on every rank."""
    from oracle import ffwd_oracle as orc
    from tests.fixtures import load_case
    c = load_case("cfg1")
    lw, pred, comp = c["lw"], c["pred"], ff.CompensatorParams(**c["comp"])
    x = torch.from_numpy(c["x"]).cuda()
    T, d = x.shape
    k = int(c["k"])
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    res0 = torch.randn((T, d), device="cuda")
    full = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], comp, device="cuda")
    want = res0.clone()
    ff.sparse_ffn_layer(x.to(torch.bfloat16), full, dp, k, out=want, residual=want)
    for n in (2, 4):
        partials = []
        for r in range(n):
            pk = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], comp, device="cuda",
                               tp_rank=r, tp_size=n)
            partials.append(ff.sparse_ffn_layer(x.to(torch.bfloat16), pk, dp, k))
        outs = [res0.clone() for _ in range(n)]
        flags = [torch.zeros(2 * n + 1, dtype=torch.int32, device="cuda") for _ in range(n)]
        _run_ranks(partials, outs, flags, outs, 1)
        for r in range(n):
            assert torch.equal(outs[r], outs[0])
        got, ref = outs[0].double(), want.double()
        rel = float((got - ref).norm() / (ref - res0.double()).norm())
        assert rel <= 5e-3, f"TP={n}: rel-L2 of the FFN part {rel:.2e}"


@pytest.mark.parametrize("n", [2, 4])
def test_overlapped_completion_of_sharded_layer(ff, n):
    """The completion overlapped with the down projection (``ffwd_ffn_layer_tp_overlap``):
    every emulated rank runs its whole layer on its own stream with the completion on a
    second stream, K3 publishing per-block tile counts the completions drain block by
    block.  Bit-exact against the sequential path (sharded layer, then the fused
    completion: same partials, same rank-order sums) on every rank, over three layers
    reusing the counters and flags."""
    from paper_2602_00397_b200.layer import layer_workspace_bytes
    from paper_2602_00397_b200.tp import sparse_ffn_layer_tp_overlap
    from tests.fixtures import load_case
    c = load_case("cfg1")
    lw, pred, comp = c["lw"], c["pred"], ff.CompensatorParams(**c["comp"])
    xb = torch.from_numpy(c["x"]).cuda().to(torch.bfloat16)
    T, d = xb.shape
    k = int(c["k"])
    dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
    res0 = torch.randn((T, d), device="cuda")
    packs = [ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], comp, device="cuda",
                           tp_rank=r, tp_size=n) for r in range(n)]
    # sequential reference: partials, then the (non-overlapped) fused completion
    partials = [ff.sparse_ffn_layer(xb, pk, dp, k) for pk in packs]
    want = [res0.clone() for _ in range(n)]
    fl = [torch.zeros(2 * n + 1, dtype=torch.int32, device="cuda") for _ in range(n)]
    _run_ranks(partials, want, fl, want, 1)

    ws = [torch.empty(layer_workspace_bytes(T, packs[r], dp.r, k, True), dtype=torch.uint8,
                      device="cuda") for r in range(n)]
    part = [torch.empty((T, d), device="cuda") for _ in range(n)]
    flags = [torch.zeros(2 * n + 1, dtype=torch.int32, device="cuda") for _ in range(n)]
    y_done = [torch.zeros(-(-T // 128), dtype=torch.int32, device="cuda") for _ in range(n)]
    main = [torch.cuda.Stream() for _ in range(n)]
    comm = [torch.cuda.Stream() for _ in range(n)]
    cur = torch.cuda.current_stream()
    for layer in (1, 2, 3):
        outs = [res0.clone() for _ in range(n)]
        xn = [torch.empty((T, d), dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        for s in main:
            s.wait_stream(cur)
        for r in range(n):
            with torch.cuda.stream(main[r]):
                sparse_ffn_layer_tp_overlap(
                    xb, packs[r], dp, k, partials=part, outs=outs, flags=flags, y_done=y_done,
                    residual=outs[r], epoch=layer, y_epoch=layer, xnexts=xn, comm_ctas=8,
                    workspace=ws[r], comm_stream=comm[r])
        for s in main:
            cur.wait_stream(s)
        torch.cuda.synchronize()
        for r in range(n):
            assert torch.equal(part[r], partials[r]), f"rank {r} partial differs"
            assert torch.equal(outs[r], want[0]), f"layer {layer}: rank {r} output differs"
            assert torch.equal(xn[r], want[0].to(torch.bfloat16))
            assert int(y_done[r].min()) == int(y_done[r].max()) == layer * (d // (256 if d % 256 == 0 else 128 if d % 128 == 0 else 64))
    for f in flags:
        assert int(f[2 * n]) == 0


def _ipc_worker(rank, world, port, q):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_00397_b200.tp import PeerBuffers
        T, d = 257, 128
        pb = PeerBuffers(T, d, "cuda:0", with_xnext=True)
        g = torch.Generator(device="cuda").manual_seed(100 + rank)
        pb.partial.copy_(torch.randn((T, d), generator=g, device="cuda"))
        res = torch.arange(T * d, device="cuda", dtype=torch.float32).reshape(T, d) * 1e-3
        pb.out.copy_(res)
        torch.cuda.synchronize()
        dist.barrier()
        out = pb.complete(pb.out).clone()
        torch.cuda.synchronize()
        parts = [None] * world
        dist.all_gather_object(parts, pb.partial.cpu())
        want = res.cpu()
        for p in parts:
            want = want + p
        q.put((rank, bool(torch.equal(out.cpu(), want)),
               bool(torch.equal(pb.xnext.cpu(), want.to(torch.bfloat16)))))
        dist.barrier()
        pb.close()
    finally:
        dist.destroy_process_group()


def _ipc_overlap_worker(rank, world, port, q):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_00397_b200 as ff
        from paper_2602_00397_b200.tp import PeerBuffers
        from tests.fixtures import load_case
        c = load_case("cfg1")
        lw, pred, comp = c["lw"], c["pred"], ff.CompensatorParams(**c["comp"])
        xb = torch.from_numpy(c["x"]).cuda().to(torch.bfloat16)
        T, d = xb.shape
        k = int(c["k"])
        dp = ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")
        pk = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], comp, device="cuda",
                           tp_rank=rank, tp_size=world)
        part = ff.sparse_ffn_layer(xb, pk, dp, k).cpu()
        parts = [None] * world
        dist.all_gather_object(parts, part)
        res0 = torch.arange(T * d, dtype=torch.float32).reshape(T, d) * 1e-4
        want = res0.clone()
        for p in parts:
            want = want + p
        pb = PeerBuffers(T, d, "cuda:0", with_xnext=True)
        ok = []
        for _ in range(2):  # counters and flags reused across layers
            pb.out.copy_(res0)
            torch.cuda.synchronize()
            dist.barrier()
            out = pb.layer_overlap(xb, pk, dp, k, residual=pb.out).clone()
            torch.cuda.synchronize()
            dist.barrier()
            ok.append(bool(torch.equal(out.cpu(), want))
                      and bool(torch.equal(pb.xnext.cpu(), want.to(torch.bfloat16))))
        q.put((rank, all(ok)))
        dist.barrier()
        pb.close()
    finally:
        dist.destroy_process_group()


def _spawn_two(target):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = sorted(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    return results


def test_peer_buffers_across_processes(ff):
    """Two processes on the one GPU: CUDA IPC handle exchange (PeerBuffers) and the fused
    completion over the mapped peer buffers."""
    assert _spawn_two(_ipc_worker) == [(0, True, True), (1, True, True)]


def test_overlapped_layer_across_processes(ff):
    """Two processes on the one GPU, TP=2 shards of the cfg1 layer: ``layer_overlap`` over
    CUDA IPC peer buffers (partials, outputs, flags and the per-block tile counters all
    mapped from the other process) equals residual + the two ranks' partials in rank
    order, bit for bit, on both ranks and over two layers."""
    assert _spawn_two(_ipc_overlap_worker) == [(0, True), (1, True)]


@pytest.mark.parametrize("collective,extra", [("rs_ag", []), ("rs_ag", ["--reduce-dtype", "bf16"]),
                                              ("allreduce", ["--skip-alt"]),
                                              ("fused", ["--skip-alt"]),
                                              ("overlap", ["--skip-alt"])])
def test_bench_tensor_parallel_paths_run(ff, collective, extra):
    """bench.py under torchrun, 2 ranks, emulated on the one GPU (gloo for the collectives,
    staged through the host where gloo has no CUDA path; both ranks time-sliced on GPU 0):
    the default N>1 line (TP over d_ffn with the sequence-parallel residual, plus the
    sequence- and data-parallel splits as extra keys) and the all-reduce / peer-memory
    completions run end to end and the JSON line is well formed.  (Timings from this
    emulation are meaningless.)"""
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
           "--config", "1b", "--layers", "2", "--steps", "2", "--warmup", "3",
           "--parallel", "tp", "--collective", collective] + extra
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=400)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "tp2"
    assert d["collective"] and d["value"] > 0
    if collective == "rs_ag" and not extra:
        assert set(d["other_splits"]) == {"sp", "dp"}
        assert all(v["ms_per_layer"] > 0 for v in d["other_splits"].values())
