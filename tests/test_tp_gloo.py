"""Tensor parallelism over d_ffn on CPU: world_size 2 with the gloo backend.

Each rank takes its shard with the product's sharding rules
(``tp.shard_host`` = what ``pack_layer`` uploads), computes its partial FFN
on the shard (the oracle stands in for the GPU kernels here), and the
product's ``tp.allreduce_partial`` sums the partials.  The result must equal
the unsharded reference FFN; the per-rank top-k lists must partition the
global selection exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ffwd_oracle as orc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_00397_b200 as ff
        from paper_2602_00397_b200 import tp
        from tests.fixtures import load_case
        c = load_case("cfg1")
        lw, pred = c["lw"], c["pred"]
        comp = ff.CompensatorParams(**c["comp"])
        gs, us, ds, cs, nid = tp.shard_host(lw["w_gate"], lw["w_up"], lw["w_down"], comp, rank,
                                            world)
        y = np.zeros_like(c["x"])
        ok_sel = True
        for j in range(c["T"] // 128):
            xb = c["x"][j * 128:(j + 1) * 128]
            if j in (0, c["T"] // 128 - 1):  # dense first / last block
                y[j * 128:(j + 1) * 128] = orc.dense_ffn(xb, gs, us, ds)
                continue
            s = orc.predictor_forward(pred["query"], pred["w1"], pred["w2"], xb)  # replicated
            g = orc.topk_indices(s, c["k"])
            loc = tp.local_selection(g, rank, world)
            ok_sel &= bool(np.array_equal(nid[loc], g[g % world == rank]))
            yb = orc.sparse_ffn_forward(xb, gs, us, ds, loc) if loc.size else 0.0
            y[j * 128:(j + 1) * 128] = yb + orc.compensator_forward(cs.w1, cs.w2, xb)
        t = torch.from_numpy(y.astype(np.float64))  # exact sum for the check
        tp.allreduce_partial(t)
        if rank == 0:
            out["y"] = t.numpy()
        out[f"sel{rank}"] = ok_sel
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_tp2_partials_allreduce_to_reference():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["sel0"] and out["sel1"]
    from tests.fixtures import load_case
    c = load_case("cfg1")
    got = out["y"][c["y_rows"]]
    # f64 partial sums of f32 shard results vs the f32 reference: f32 rounding only
    np.testing.assert_allclose(got, c["y"], rtol=0, atol=2e-5)


def _sp_worker(rank, world, port, out):
    """Sequence parallelism: each rank runs the engine's FFN branch (oracle) on its
    contiguous share of the prompt's blocks (``layer.seq_shard``), dense only where it
    holds the prompt's first / last block; no collective on the data path -- the shards
    are gathered here only to check them."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_00397_b200 as ff
        from paper_2602_00397_b200.layer import seq_shard
        from tests.fixtures import load_case
        c = load_case("cfg1")
        lw, pred = c["lw"], c["pred"]
        comp = ff.CompensatorParams(**c["comp"])
        n_blk = c["T"] // 128
        b0, b1, dfl = seq_shard(n_blk, rank, world)
        y = np.zeros((c["T"], c["x"].shape[1]), dtype=np.float32)
        for i, j in enumerate(range(b0, b1)):
            xb = c["x"][j * 128:(j + 1) * 128]
            dense = (i == 0 and dfl in (True, "first")) or (j == b1 - 1 and dfl in (True, "last"))
            if dense:
                y[j * 128:(j + 1) * 128] = orc.dense_ffn(xb, lw["w_gate"], lw["w_up"], lw["w_down"])
                continue
            s = orc.predictor_forward(pred["query"], pred["w1"], pred["w2"], xb)
            g = orc.topk_indices(s, c["k"])
            y[j * 128:(j + 1) * 128] = (orc.sparse_ffn_forward(xb, lw["w_gate"], lw["w_up"],
                                                              lw["w_down"], g)
                                        + orc.compensator_forward(comp.w1, comp.w2, xb))
        parts = [None] * world
        dist.all_gather_object(parts, (b0, b1, y[b0 * 128:b1 * 128]))
        if rank == 0:
            out["parts"] = parts
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sp2_shards_tile_the_prompt_and_match_reference():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sp_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from tests.fixtures import load_case
    c = load_case("cfg1")
    parts = sorted(out["parts"], key=lambda p: p[0])
    n_blk = c["T"] // 128
    assert parts[0][0] == 0 and parts[-1][1] == n_blk
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))  # contiguous, disjoint
    y = np.concatenate([p[2] for p in parts])
    np.testing.assert_allclose(y[c["y_rows"]], c["y"], rtol=0, atol=2e-5)


def test_seq_shard_rules():
    from paper_2602_00397_b200.errors import ValidationError
    from paper_2602_00397_b200.layer import seq_shard
    assert seq_shard(128, 0, 1) == (0, 128, True)
    assert [seq_shard(128, r, 4) for r in range(4)] == [
        (0, 32, "first"), (32, 64, False), (64, 96, False), (96, 128, "last")]
    assert [seq_shard(10, r, 3)[:2] for r in range(3)] == [(0, 3), (3, 6), (6, 10)]
    with pytest.raises(ValidationError):
        seq_shard(2, 0, 4)
    from paper_2602_00397_b200.layer import dense_first_last_code
    assert [dense_first_last_code(v) for v in (False, True, "first", "last")] == [0, 1, 2, 3]
    assert dense_first_last_code(1) == 1 and dense_first_last_code(0) == 0
    with pytest.raises(ValidationError):
        dense_first_last_code("middle")
