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
