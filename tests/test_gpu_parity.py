"""GPU parity: the sm_100a path against the oracle / the reference's golden vectors.

Bar:
  * predictor scores and selected indices: bit-exact;
  * FFN outputs (bf16 operands, f32 accumulation, bf16 hidden):
        rel-L2 <= 5e-3   and   max|diff| <= 3e-2 * rms(y_ref).
"""

import numpy as np
import pytest
import torch

from oracle import ffwd_oracle as orc
from tests.fixtures import golden, load_case

pytestmark = pytest.mark.gpu

REL_L2 = 5e-3
MAX_REL_RMS = 3e-2


@pytest.fixture(scope="module")
def ff():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_00397_b200 as ff
    from paper_2602_00397_b200 import _lib
    _lib.require_device(torch.cuda.current_device())
    return ff


def assert_close(got, want, what=""):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    rms = np.sqrt((want ** 2).mean())
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    mx = np.abs(got - want).max() / max(rms, 1e-30)
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    assert rel <= REL_L2, f"{what}: rel-L2 {rel:.3e} > {REL_L2}"
    assert mx <= MAX_REL_RMS, f"{what}: max|d|/rms {mx:.3e} > {MAX_REL_RMS}"
    return rel, mx


def dev_pred(ff, pred):
    return ff.DevicePredictor.from_params(ff.PredictorParams(**pred), "cuda")


@pytest.mark.parametrize("name", ["tiny_dfl", "tiny_all", "tiny_k25", "cfg1", "l1b", "l8b_pred",
                                  "qwen8b_pred"])
def test_predictor_scores_and_indices_bit_exact(ff, name):
    c = load_case(name)
    dp = dev_pred(ff, c["pred"])
    for dtype in (torch.bfloat16, torch.float32):
        x = torch.from_numpy(c["x"]).to("cuda", dtype)
        sb = c["sparse_blocks"]
        if sb.size == 0:
            continue
        assert (np.diff(sb) == 1).all()
        s = ff.predictor_scores(dp, x, int(sb[0]), int(sb.size))
        got = s.cpu().numpy()
        np.testing.assert_array_equal(got.view(np.uint32), c["scores"].view(np.uint32))
        from paper_2602_00397_b200.sparse import topk_device
        idx = topk_device(s, c["k"]).cpu().numpy()
        np.testing.assert_array_equal(idx, c["indices"])


@pytest.mark.parametrize("d,r,f,n_blk", [(256, 16, 1376, 1), (1024, 64, 3000, 31),
                                          (2048, 128, 4096, 33), (4096, 256, 2048, 64),
                                          (1000, 64, 2500, 7), (2048, 128, 8192, 65)])
def test_predictor_short_prompt_paths_bit_exact(ff, d, r, f, n_blk):
    """The predictor GEMM paths of short prompts (<= 64 blocks: W1's split-K summed in a
    thread-block cluster, 32- / 64-row tiles, the h-resident scores GEMM from 4096 columns)
    and their neighbours (65 blocks: the 128-row split-K path): scores bit-identical to the
    oracle (predictor.py:68-81) for every block, both input dtypes, odd d / r / f / counts."""
    rng = np.random.default_rng(d + r + f + n_blk)
    pred = orc.init_predictor(rng, d, f, r)
    T = 128 * n_blk - 37 if n_blk > 1 else 128  # a short tail block
    x = orc.bf16_round(rng.standard_normal((T, d)).astype(np.float32))
    dp = dev_pred(ff, pred)
    want = np.stack([orc.predictor_forward(pred["query"], pred["w1"], pred["w2"],
                                           x[128 * b:min(T, 128 * b + 128)])
                     for b in range(n_blk)])
    for dtype in (torch.bfloat16, torch.float32):
        got = ff.predictor_scores(dp, torch.from_numpy(x).to("cuda", dtype)).cpu().numpy()
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32),
                                      err_msg=f"{dtype}")


def test_topk_edge_cases_match_reference(ff):
    from paper_2602_00397_b200.sparse import topk_device
    g = golden("topk_edges")
    for i, k in enumerate(g["k"]):
        s = g["scores"][g["offs_s"][i]:g["offs_s"][i + 1]]
        want = g["indices"][g["offs_i"][i]:g["offs_i"][i + 1]]
        got = topk_device(torch.from_numpy(s.copy()).cuda(), int(k))[0].cpu().numpy()
        np.testing.assert_array_equal(got, want, err_msg=f"case {i}")


def test_topk_large_random_rows(ff):
    from paper_2602_00397_b200.sparse import topk_device
    rng = np.random.default_rng(3)
    for f, k in [(14336, 7168), (12288, 4547), (8192, 2048), (1376, 688), (65536, 1000)]:
        s = rng.standard_normal((4, f)).astype(np.float32)
        s[1] = np.round(s[1] * 4) / 4  # many ties
        s[2, ::7] = -0.0
        s[3, ::11] = np.nan
        got = topk_device(torch.from_numpy(s).cuda(), k).cpu().numpy()
        for r in range(4):
            np.testing.assert_array_equal(got[r], orc.topk_indices(s[r], k))


def test_topk_tp_local_lists(ff):
    from paper_2602_00397_b200 import _dev, _lib
    rng = np.random.default_rng(4)
    f, k = 14336, 7168
    s = rng.standard_normal((3, f)).astype(np.float32)
    st = torch.from_numpy(s).cuda()
    lib = _dev.lib_for(st.device)
    for tp in (2, 4, 8):
        for rank in range(tp):
            loc = torch.full((3, k), -1, dtype=torch.int32, device="cuda")
            cnt = torch.zeros(3, dtype=torch.int32, device="cuda")
            _lib.check(lib.ffwd_topk(st.data_ptr(), 3, f, k, rank, tp, None, 0, loc.data_ptr(), k,
                                     cnt.data_ptr(), _dev.stream_handle(st.device)), "topk")
            loc, cnt = loc.cpu().numpy(), cnt.cpu().numpy()
            for r in range(3):
                full = orc.topk_indices(s[r], k)
                mine = full[full % tp == rank] // tp
                assert cnt[r] == mine.size
                np.testing.assert_array_equal(loc[r, :cnt[r]], mine)


def test_topk_widths_ties_and_tp(ff):
    """Top-k over rows of 2K-32K scores: widths that are not multiples of the thread count,
    ties spread over the whole row (one giant tie, duplicated halves, -0 / NaN), k at
    1 / f-1 / f, and the global list plus the rank-local lists + counts under TP."""
    from paper_2602_00397_b200 import _dev, _lib
    rng = np.random.default_rng(11)
    for f in (2048, 2052, 4100, 8192, 12288, 14336, 30000, 32768):
        rows = 5
        s = rng.standard_normal((rows, f)).astype(np.float32)
        s[1] = np.round(s[1] * 2) / 2          # few distinct values: ties across chunks
        s[2] = 0.0                              # one giant tie
        s[2, ::5] = -0.0
        s[3, ::3] = np.nan
        s[4, f // 2:] = s[4, :f - f // 2]       # duplicated halves
        st = torch.from_numpy(s).cuda()
        lib = _dev.lib_for(st.device)
        for k in (1, 7, f // 3, f // 2, f - 1, f):
            for tp, rank in ((1, 0), (2, 1), (8, 5)):
                kl = min(k, (f + tp - 1) // tp)
                glob = torch.full((rows, k), -1, dtype=torch.int32, device="cuda")
                loc = torch.full((rows, kl), -1, dtype=torch.int32, device="cuda")
                cnt = torch.zeros(rows, dtype=torch.int32, device="cuda")
                _lib.check(lib.ffwd_topk(st.data_ptr(), rows, f, k, rank, tp, glob.data_ptr(), k,
                                         loc.data_ptr(), kl, cnt.data_ptr(),
                                         _dev.stream_handle(st.device)), "topk")
                g, lc, c = glob.cpu().numpy(), loc.cpu().numpy(), cnt.cpu().numpy()
                for r in range(rows):
                    full = orc.topk_indices(s[r], k)
                    np.testing.assert_array_equal(g[r], full, err_msg=f"f={f} k={k} row {r}")
                    mine = full[full % tp == rank] // tp
                    assert c[r] == mine.size, (f, k, tp, r)
                    np.testing.assert_array_equal(lc[r, :c[r]], mine)


def _layer_case(ff, name):
    c = load_case(name)
    lw = c["lw"]
    comp = ff.CompensatorParams(**c["comp"])
    packed = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], comp, device="cuda")
    return c, packed, dev_pred(ff, c["pred"])


@pytest.mark.parametrize("name", ["tiny_dfl", "tiny_all", "tiny_k25", "cfg1", "l1b"])
def test_ffn_layer_matches_reference(ff, name):
    c, packed, dp = _layer_case(ff, name)
    x = torch.from_numpy(c["x"]).to("cuda", torch.bfloat16)
    y, idx = ff.sparse_ffn_layer(x, packed, dp, c["k"], dense_first_last=c["dense_first_last"],
                                 return_indices=True)
    torch.cuda.synchronize()
    if c["sparse_blocks"].size:
        np.testing.assert_array_equal(idx.cpu().numpy(), c["indices"])
    y = y.cpu().numpy()
    got = y[c["y_rows"]] if "y_rows" in c else y
    assert_close(got, c["y"], name)


def test_dense_layer_and_full_k_shortcut(ff):
    c, packed, dp = _layer_case(ff, "cfg1")
    x = torch.from_numpy(c["x"]).to("cuda", torch.bfloat16)
    lw = c["lw"]
    want = orc.dense_ffn(c["x"], lw["w_gate"], lw["w_up"], lw["w_down"])
    assert_close(ff.dense_ffn(x, packed).cpu().numpy(), want, "dense_ffn")
    # k == d_ffn: every block dense, no predictor, no compensator (engine.py:268)
    y = ff.sparse_ffn_layer(x, packed, dp, c["f"], dense_first_last=True)
    assert_close(y.cpu().numpy(), want, "full-k layer")


def test_full_mask_is_bit_identical_to_dense(ff):
    """Acceptance criterion 1's second half (test_sparse.py:107-115): the gathered FFN
    with every neuron selected equals the dense FFN bit for bit -- the gather4 path
    (explicit ascending index) and the 2-D tile path (identity) stage identical bytes."""
    c, packed, _ = _layer_case(ff, "cfg1")
    x = torch.from_numpy(c["x"]).to("cuda", torch.bfloat16)
    f = c["f"]
    n_blk = -(-x.shape[0] // 128)
    ld = -(-f // 4) * 4
    idx = torch.zeros((n_blk, ld), dtype=torch.int32, device="cuda")
    idx[:, :f] = torch.arange(f, dtype=torch.int32, device="cuda")
    y_gather = ff.run_sparse_ffn(x, packed, idx, f, has_comp=False)
    y_dense = ff.dense_ffn(x, packed)
    assert torch.equal(y_gather, y_dense)


def test_reference_api_drop_in(ff):
    """predictor_forward / build_mask / select_subweights / sparse_ffn_forward /
    compensator_forward with numpy in, numpy out (engine.py:286-300 call pattern)."""
    c = load_case("cfg1")
    lw = ff.LayerWeights(w_gate=c["lw"]["w_gate"], w_up=c["lw"]["w_up"],
                         w_down=c["lw"]["w_down"])
    pred = ff.PredictorParams(**c["pred"])
    comp = ff.CompensatorParams(**c["comp"])
    j = int(c["sparse_blocks"][2])
    xb = c["x"][j * 128:(j + 1) * 128]
    s = ff.predictor_forward(pred, xb)
    assert isinstance(s, np.ndarray) and s.dtype == np.float32
    np.testing.assert_array_equal(s.view(np.uint32), c["scores"][2].view(np.uint32))
    mask = ff.build_mask(s, c["k"], layer=0, block=j)
    np.testing.assert_array_equal(mask.indices, c["indices"][2])
    sub = ff.select_subweights(lw, mask)
    y = ff.sparse_ffn_forward(xb, sub)
    want_ffn = orc.sparse_ffn_forward(xb, lw.w_gate, lw.w_up, lw.w_down, mask.indices)
    assert_close(y, want_ffn, "sparse_ffn_forward")
    corr = ff.compensator_forward(comp, xb)
    want_c = orc.compensator_forward(comp.w1, comp.w2, xb)
    assert_close(corr, want_c, "compensator_forward")
    yc = ff.apply_compensation(y, corr)
    rows = c["y_rows"]
    sel = (rows >= j * 128) & (rows < (j + 1) * 128)
    assert_close(yc[rows[sel] - j * 128], c["y"][sel], "sparse + compensation vs reference")


def test_tensor_parallel_shards_sum_to_full(ff):
    """TP over d_ffn emulated on one GPU: per-rank partials sum to the TP=1 result."""
    c = load_case("cfg1")
    lw, comp = c["lw"], ff.CompensatorParams(**c["comp"])
    dp = dev_pred(ff, c["pred"])
    x = torch.from_numpy(c["x"]).to("cuda", torch.bfloat16)
    full_p = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], comp, device="cuda")
    y1, i1 = ff.sparse_ffn_layer(x, full_p, dp, c["k"], return_indices=True)
    for tp in (2, 4, 8):
        acc = torch.zeros_like(y1)
        for rank in range(tp):
            p = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], comp, device="cuda",
                              tp_rank=rank, tp_size=tp)
            yr, ir = ff.sparse_ffn_layer(x, p, dp, c["k"], return_indices=True)
            assert torch.equal(ir, i1)
            acc += yr
        assert_close(acc.cpu().numpy(), y1.cpu().numpy(), f"tp{tp}")
        rows = c["y_rows"]
        assert_close(acc.cpu().numpy()[rows], c["y"], f"tp{tp} vs reference")


def test_errors_map_to_reference_types(ff):
    c, packed, dp = _layer_case(ff, "tiny_all")
    x = torch.from_numpy(c["x"]).to("cuda", torch.bfloat16)
    with pytest.raises(ff.ValidationError):
        ff.sparse_ffn_layer(x, packed, dp, 0)
    with pytest.raises(ff.ValidationError):
        ff.sparse_ffn_layer(x, packed, dp, c["f"] + 1)
    with pytest.raises(ff.ValidationError):
        ff.topk_indices(np.ones(3, np.float32), 4)
    # any d_model works on the per-block drop-ins (zero-padded to the 64-column atom) ...
    rng = np.random.default_rng(96)
    w = {n_: orc.bf16_round(rng.standard_normal(s_).astype(np.float32) * np.float32(0.1))
         for n_, s_ in (("g", (96, 200)), ("u", (96, 200)), ("dn", (200, 96)))}
    p96 = ff.pack_layer(w["g"], w["u"], w["dn"], None, device="cuda")
    x96 = orc.bf16_round(rng.standard_normal((128, 96)).astype(np.float32))
    got = ff.dense_ffn(torch.from_numpy(x96).cuda(), p96).cpu().numpy()
    assert got.shape == (128, 96)
    assert_close(got, orc.dense_ffn(x96, w["g"], w["u"], w["dn"]), "d=96 dense drop-in")
    # ... but the layer-batched hot path keeps the kernels' native width
    dp96 = ff.DevicePredictor.from_params(
        ff.PredictorParams(**orc.init_predictor(rng, 96, 200)), "cuda")
    with pytest.raises(ff.UnsupportedError):
        ff.sparse_ffn_layer(torch.zeros((128, 96), device="cuda"), p96, dp96, 100)


@pytest.mark.parametrize("shape", [("l8b", 4096, 14336), ("qwen8b", 4096, 12288)])
def test_full_size_properties(ff, shape):
    """BASELINE-size layer (T=16K / 8K): sampled blocks vs the oracle, plus
    size-independent properties (sorted unique indices, finite outputs)."""
    name, d, f = shape
    T = 16384 if name == "l8b" else 8192
    k = orc.budget_to_k(0.5, f)
    rng = np.random.default_rng(77)
    lw = orc.random_layer(rng, d, f, 0.02)
    pred = orc.init_predictor(np.random.default_rng([77, 0]), d, f)
    comp = {k_: orc.bf16_round(v) for k_, v in
            orc.init_compensator(np.random.default_rng([78, 0]), d).items()}
    for key in ("w_gate", "w_up", "w_down"):
        lw[key] = orc.bf16_round(lw[key])
    xg = torch.randn((T, d), generator=torch.Generator().manual_seed(5)).to(torch.bfloat16)
    x_np = xg.float().numpy()
    packed = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], ff.CompensatorParams(**comp),
                           device="cuda")
    dp = dev_pred(ff, pred)
    y, idx = ff.sparse_ffn_layer(xg.cuda(), packed, dp, k, return_indices=True)
    # determinism across back-to-back launches (programmatic dependent launch, the
    # block-granular K2 -> K3 counters and the CTA-pair multicast must not race)
    res = torch.randn((T, d), device="cuda")
    outs = []
    for _ in range(3):
        o = res.clone()
        ff.sparse_ffn_layer(xg.cuda(), packed, dp, k, out=o, residual=o)
        outs.append(o)
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:]), "non-deterministic layer output"
    assert torch.equal(outs[0] - res, outs[0] - res)  # finite
    assert torch.allclose(outs[0] - res, y, rtol=0, atol=1e-5 * float(y.abs().max()))
    idx = idx.cpu().numpy()
    y = y.cpu().numpy()
    assert np.isfinite(y).all()
    assert (np.diff(idx, axis=1) > 0).all() and idx.min() >= 0 and idx.max() < f
    n_blk = T // 128
    for j in (1, n_blk // 2, n_blk - 2):
        xb = x_np[j * 128:(j + 1) * 128]
        s = orc.predictor_forward(pred["query"], pred["w1"], pred["w2"], xb)
        want_idx = orc.topk_indices(s, k)
        np.testing.assert_array_equal(idx[j - 1], want_idx)
    for j in (0, n_blk // 2):  # one dense first block, one predicted block
        xb = x_np[j * 128:(j + 1) * 128]
        if j == 0:
            want = orc.dense_ffn(xb, lw["w_gate"], lw["w_up"], lw["w_down"])
        else:
            want = orc.sparse_ffn_forward(xb, lw["w_gate"], lw["w_up"], lw["w_down"], idx[j - 1])
            want = want + orc.compensator_forward(comp["w1"], comp["w2"], xb)
        assert_close(y[j * 128:(j + 1) * 128], want, f"{name} block {j}")


@pytest.mark.parametrize("d,f,T,k,dfl", [
    (192, 520, 1, 17, True),      # one token, one (dense) block
    (192, 520, 129, 259, True),   # second block holds one token; both dense
    (192, 520, 300, 1, False),    # k = 1; 64-column down tiles (d % 128 != 0)
    (192, 520, 300, 519, False),  # k = f - 1; odd up-tile counts (CTA-pair repeats)
    (320, 1000, 400, 333, True),  # odd column-tile count in K3, ragged compensator
    (256, 768, 640, 768, True),   # k == f: full-K shortcut, every block dense
])
def test_layer_edge_shapes_vs_oracle(ff, d, f, T, k, dfl):
    """Edge shapes of the reference's own tests (short / single-token blocks, k = 1,
    k = f - 1, k = f) and of this build's tiling (64/128-column down tiles, odd tile
    counts under CTA pairs, ragged compensator): indices bit-exact, outputs in tolerance."""
    rng = np.random.default_rng(d * 7 + T)
    lw = orc.random_layer(rng, d, f, 0.02)
    for key in ("w_gate", "w_up", "w_down"):
        lw[key] = orc.bf16_round(lw[key])
    pred = orc.init_predictor(np.random.default_rng([d, T]), d, f)
    comp = {k_: orc.bf16_round(v) for k_, v in
            orc.init_compensator(np.random.default_rng([d, T, 1]), d).items()}
    x = orc.bf16_round(rng.standard_normal((T, d)).astype(np.float32))
    packed = ff.pack_layer(lw["w_gate"], lw["w_up"], lw["w_down"], ff.CompensatorParams(**comp),
                           device="cuda")
    dp = dev_pred(ff, pred)
    y, idx = ff.sparse_ffn_layer(torch.from_numpy(x).to("cuda", torch.bfloat16), packed, dp, k,
                                 dense_first_last=dfl, return_indices=True)
    torch.cuda.synchronize()
    want, masks, _ = orc.ffn_layer_blockwise(x, lw, pred, comp, k, dfl, keep_masks=True)
    if masks:
        got = idx.cpu().numpy()
        for row, j in enumerate(sorted(masks)):
            np.testing.assert_array_equal(got[row], masks[j])
    assert_close(y.cpu().numpy(), want, f"d{d} f{f} T{T} k{k}")


def test_scores_gemm_paths_agree_bit_exactly(ff):
    """The scores GEMM (predictor.py:80) runs on the h-resident kernel for <= 64 predicted
    blocks and on 16-column tiles above: the same block gives bit-identical scores either
    way, and both match the oracle bit for bit (8B predictor shape)."""
    from oracle import ffwd_oracle as orc
    d, r, f = 4096, 256, 14336
    rng = np.random.default_rng(11)
    q = (rng.standard_normal((1, d)) * 0.02).astype(np.float32)
    w1 = (rng.standard_normal((d, r)) * 0.02).astype(np.float32)
    w2 = (rng.standard_normal((r, f)) * 0.02).astype(np.float32)
    dp = ff.DevicePredictor(query=torch.from_numpy(q[0]).cuda(), w1=torch.from_numpy(w1).cuda(),
                            w2=torch.from_numpy(w2).cuda())
    x = torch.randn((126 * 128, d), device="cuda").to(torch.bfloat16).float()
    from paper_2602_00397_b200.predictor import predictor_scores
    full = predictor_scores(dp, x)                       # 126 blocks: tiled kernel
    for n in (14, 40, 62):                               # resident kernel, 1 and 2 row groups
        part = predictor_scores(dp, x[:n * 128])
        assert torch.equal(part, full[:n]), f"{n} blocks: scores differ from the tiled path"
    xs = x.cpu().numpy()
    for b in (0, 13, 61, 125):
        want = orc.predictor_forward(q, w1, w2, xs[b * 128:(b + 1) * 128])
        assert np.array_equal(full[b].cpu().numpy(), want), f"block {b} differs from the oracle"
