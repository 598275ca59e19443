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


def _rms_bf16(h, gain, eps=1e-6):  # kernels.py:96-106, then the bf16 FFN operand
    h64 = h.astype(np.float64)
    scale = 1.0 / np.sqrt((h64 * h64).mean(axis=1, keepdims=True) + eps)
    return orc.bf16_round((h64 * scale * gain.astype(np.float64)).astype(np.float32))


def _sp_tp_model(d=512, f=1376, L=2, seed=31):
    layers = []
    for l in range(L):
        lw = orc.random_layer(np.random.default_rng([seed, l]), d, f, 0.02)
        lw = {k: orc.bf16_round(lw[k]) for k in ("w_gate", "w_up", "w_down")}
        pred = orc.init_predictor(np.random.default_rng([seed, l, 1]), d, f)
        comp = {k: orc.bf16_round(v) for k, v in
                orc.init_compensator(np.random.default_rng([seed, l, 2]), d).items()}
        layers.append((lw, pred, comp, orc.budget_to_k(0.5, f)))
    return layers


def _ffn_blocks(x, lw, pred, comp, k, nid=None, rank=0, world=1, given=None):
    """The engine's FFN branch over all blocks of x (engine.py:254-310), on the neuron
    shard `nid` (strided, rank of world) when given; returns (y, global index rows).
    `given` {block: global index row} replaces the predictor (a gathered selection)."""
    T = x.shape[0]
    n_blk = T // 128
    y = np.zeros_like(x)
    sel = {}
    gs, us, ds = lw["w_gate"], lw["w_up"], lw["w_down"]
    c1, c2 = comp["w1"], comp["w2"]
    if nid is not None:
        gs, us, ds = gs[:, nid], us[:, nid], ds[nid]
        from paper_2602_00397_b200.layer import shard_comp_cols
        lo, hi = shard_comp_cols(c1.shape[1], rank, world)
        c1, c2 = c1[:, lo:hi], c2[lo:hi]
    for j in range(n_blk):
        xb = x[j * 128:(j + 1) * 128]
        if j in (0, n_blk - 1):
            y[j * 128:(j + 1) * 128] = orc.dense_ffn(xb, gs, us, ds)
            continue
        if given is not None:
            g = given[j]
        else:
            s = orc.predictor_forward(pred["query"], pred["w1"], pred["w2"], xb)
            g = orc.topk_indices(s, k)
        sel[j] = g
        loc = g if nid is None else g[g % world == rank] // world
        yb = orc.sparse_ffn_forward(xb, gs, us, ds, loc) if loc.size else 0.0
        y[j * 128:(j + 1) * 128] = yb + (orc.compensator_forward(c1, c2, xb) if c1.shape[1]
                                         else 0.0)
    return y, sel


def _pack_mask(rows, f):
    """Selection bitmasks (layer.predict_mask's format) of index rows, int32 words."""
    m = np.zeros((len(rows), (f + 31) // 32), np.uint32)
    for i, g in enumerate(rows):
        np.bitwise_or.at(m[i], g >> 5, (np.uint32(1) << (g & 31).astype(np.uint32)))
    return m.view(np.int32)


def _sp_tp_worker(rank, world, port, out, sharded=False):
    """SeqParallelTP with gloo collectives and the oracle in place of the kernels: each
    rank owns T/N residual rows, normalises them, all-gathers x and the logits, runs the
    FFN branch on its strided d_ffn shard, reduce-scatters the partial y.  `sharded`:
    the sequence-parallel predictor -- each rank predicts its own blocks, the ranks
    all-gather the selection bitmasks instead of the logits."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_00397_b200.layer import shard_neurons
        from paper_2602_00397_b200.tp import SeqParallelTP, TorchComm, seq_rows
        model = _sp_tp_model()
        d, f, T = 512, 1376, 1024
        gain = np.ones(d, np.float32)
        h0 = orc.bf16_round(np.random.default_rng(5).standard_normal((T, d)).astype(np.float32))
        r0, r1 = seq_rows(T, rank, world)
        nid = shard_neurons(f, rank, world)
        log = {"sel_ok": True, "lg_ok": True, "predicted": 0}

        def norm_fn(l, h_shard, add):
            if add is not None:
                h_shard.add_(add)  # engine.py:308 then :267
            x = _rms_bf16(h_shard.numpy(), gain)
            sp.x_shard.copy_(torch.from_numpy(x))
            q = model[l][1]["query"]
            sp.lg_shard.copy_(torch.from_numpy(orc.mm(q, x.T)[0] / np.float32(np.sqrt(d))))

        def predict_fn(l, lo, hi):  # this rank's own blocks -> bitmask rows
            _, pred, _, k = model[l]
            x = sp.x_shard.numpy()
            rows = [orc.topk_indices(orc.predictor_forward(pred["query"], pred["w1"], pred["w2"],
                                                           x[b * 128:(b + 1) * 128]), k)
                    for b in range(lo, hi)]
            sp.mask_shard[lo:hi].copy_(torch.from_numpy(_pack_mask(rows, f)))
            log["predicted"] += hi - lo

        def ffn_fn(l, x_full, sel_full, y_part):
            lw, pred, comp, k = model[l]
            x = x_full.numpy()
            _, want_sel = _ffn_blocks(x, lw, pred, comp, k)
            given = None
            if sharded:  # the gathered bitmasks are every block's global selection
                m = sel_full.numpy().view(np.uint32)
                bits = np.unpackbits(m.view(np.uint8), axis=1, bitorder="little")[:, :f]
                given = {j: np.flatnonzero(bits[j]) for j in want_sel}
            else:
                want_lg = orc.mm(pred["query"], x.T)[0] / np.float32(np.sqrt(d))
                log["lg_ok"] &= bool(np.array_equal(sel_full.numpy(), want_lg))
            y, sel = _ffn_blocks(x, lw, pred, comp, k, nid, rank, world, given=given)
            log["sel_ok"] &= all(np.array_equal(sel[j], want_sel[j]) for j in want_sel)
            y_part.copy_(torch.from_numpy(y))

        sp = SeqParallelTP([(None, None, k) for _, _, _, k in model], T, d, rank, world, "cpu",
                           comm=TorchComm(), norm_fn=norm_fn, ffn_fn=ffn_fn,
                           predict_fn=predict_fn, x_dtype=torch.float32,
                           shard_predictor=sharded, f=f)
        h = torch.from_numpy(h0[r0:r1].copy())
        sp.stack(h)
        parts = [None] * world
        dist.all_gather_object(parts, (r0, h.numpy(), log))
        if rank == 0:
            out["parts"] = parts
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("sharded", [False, True], ids=["replicated_predictor",
                                                       "sharded_predictor"])
def test_sp_tp2_reduce_scatter_all_gather_matches_reference(sharded):
    """World 2: the sequence-parallel TP stack (reduce-scatter / all-gather around the
    FFN branch, engine.py:263-308 split over d_ffn and over the residual rows) equals the
    unsharded reference chain h <- h + FFN(rmsnorm(h)) over two layers.  Sharded: each
    rank predicts only its own blocks (4 of the 8; the dense first / last excluded) and
    the gathered bitmasks equal every block's global selection."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sp_tp_worker, args=(2, _free_port(), out, sharded), nprocs=2, join=True)
    parts = sorted(out["parts"], key=lambda p: p[0])
    assert all(p[2]["sel_ok"] and p[2]["lg_ok"] for p in parts)
    # layers x own predicted blocks: rank 0 skips block 0, rank 1 block 7
    assert [p[2]["predicted"] for p in parts] == ([2 * 3, 2 * 3] if sharded else [0, 0])
    h_tp = np.concatenate([p[1] for p in parts])
    d, T = 512, 1024
    h = orc.bf16_round(np.random.default_rng(5).standard_normal((T, d)).astype(np.float32))
    for lw, pred, comp, k in _sp_tp_model():
        y, _ = _ffn_blocks(_rms_bf16(h, np.ones(d, np.float32)), lw, pred, comp, k)
        h = h + y
    rel = np.linalg.norm(h_tp - h) / np.linalg.norm(h)
    assert rel < 1e-5, rel  # f32 partial sums vs one accumulation: rounding only


def test_sharded_predictor_block_ranges():
    """SeqParallelTP.predicted_blocks: each rank predicts exactly its own blocks minus the
    prompt's dense first / last block (engine.py:258-262), none under the full-K shortcut
    (engine.py:268), and the ranks' ranges tile the predicted blocks."""
    from paper_2602_00397_b200.errors import ValidationError
    from paper_2602_00397_b200.tp import SeqParallelTP
    T, d, f = 2048, 64, 256
    n_blk = T // 128
    for world in (1, 2, 4, 8):
        for dfl in (True, False):
            got = []
            for rank in range(world):
                sp = SeqParallelTP([(None, None, 128)], T, d, rank, world, "cpu", comm=None,
                                   norm_fn=lambda *a: None, ffn_fn=lambda *a: None,
                                   predict_fn=lambda *a: None, shard_predictor=True, f=f,
                                   dense_first_last=dfl, x_dtype=torch.float32)
                lo, hi = sp.predicted_blocks(128)
                nbr = n_blk // world
                got += [rank * nbr + b for b in range(lo, hi)]
                assert sp.predicted_blocks(f) == (0, 0)  # k == d_ffn: every block dense
            want = list(range(1, n_blk - 1)) if dfl else list(range(n_blk))
            assert got == want, (world, dfl, got)
    with pytest.raises(ValidationError):  # rows must be whole blocks per rank
        SeqParallelTP([(None, None, 128)], 1024, d, 0, 16, "cpu", comm=None,
                      shard_predictor=True, f=f, x_dtype=torch.float32)
