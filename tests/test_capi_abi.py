"""C-ABI boundary checks that need no GPU: the library loads, exports and binds
every entry point include/ffwd_b200.h declares, host-only entry points work,
and compute entry points fail loudly (no CPU fallback) when there is no GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2602_00397_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ffwd_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FFWD_API\s+[\w\s\*]+?\b(ffwd_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    assert {"ffwd_ffn_layer", "ffwd_predictor_forward", "ffwd_topk", "ffwd_sparse_ffn",
            "ffwd_predict_topk", "ffwd_layer_workspace_bytes"} <= set(syms)


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_abi_version_and_host_only_calls():
    lib = _lib.load_library()
    assert lib.ffwd_abi_version() == 1
    # workspace sizing is pure host arithmetic
    ws = lib.ffwd_layer_workspace_bytes(16384, 4096, 14336, 14336, 512, 256, 7168, 1, 1)
    h_bytes = 128 * 128 * 14336 * 2  # H for 128 blocks at the dense width
    assert h_bytes < ws < h_bytes + 64 * 2 ** 20
    assert lib.ffwd_predictor_workspace_bytes(126, 4096, 256, 14336) > 126 * 4096 * 4
    assert lib.ffwd_sparse_ffn_workspace_bytes(1024, 512, 1376, 64, 688) > 0
    assert lib.ffwd_set_raster(32, 8) == _lib.FFWD_OK
    assert lib.ffwd_set_raster(0, 8) == _lib.FFWD_ERR_VALIDATION
    assert b"raster" in lib.ffwd_last_error()
    for i in range(7):
        assert lib.ffwd_stage_name(i)


def test_validation_happens_before_any_launch():
    lib = _lib.load_library()
    # k out of range -> FFWD_ERR_VALIDATION (ValidationError), no device touched
    rc = lib.ffwd_topk(None, 1, 10, 11, 0, 1, None, 0, None, 0, None, None)
    assert rc == _lib.FFWD_ERR_VALIDATION
    with pytest.raises(_lib.ValidationError):
        _lib.check(rc, "topk")
    rc = lib.ffwd_topk(None, 1, 10, 5, 3, 2, None, 0, None, 0, None, None)
    assert rc == _lib.FFWD_ERR_VALIDATION and b"rank" in lib.ffwd_last_error()
    rc = lib.ffwd_ffn_layer(None, 256, 96, None, None, 200, 12, None, None, None, 8, 200, 100, 1,
                            1, 0, 1, None, None, None, None, 0, None, 0, None)
    assert rc == _lib.FFWD_ERR_UNSUPPORTED  # d_model % 64 != 0
    with pytest.raises(_lib.UnsupportedError):
        _lib.check(rc, "ffn_layer")
    # dense_first_last codes: 0..3 (3 = a sequence shard holding the prompt's last block)
    args = [None, 256, 512, None, None, 1376, 64, None, None, None, 32, 1376, 688]
    tail = [1, 0, 1, None, None, None, None, 0, None, None, None, 0, None]
    assert lib.ffwd_ffn_layer2(*args, 5, *tail) == _lib.FFWD_ERR_VALIDATION
    assert b"dense_first_last" in lib.ffwd_last_error()
    # the overlapped TP layer rejects missing peer buffers before touching the device
    rc = lib.ffwd_ffn_layer_tp_overlap(None, 256, 512, None, None, 688, 32, None, None, None,
                                       32, 1376, 688, 1, 1, 0, 2, None, 0, None, None, None,
                                       None, None, None, None, None, 1, 1, 0, None, 0, None,
                                       None)
    assert rc == _lib.FFWD_ERR_VALIDATION and b"pointers" in lib.ffwd_last_error()
    rc = lib.ffwd_ffn_layer_tp_overlap(None, 256, 512, None, None, 688, 32, None, None, None,
                                       32, 1376, 688, 1, 1, 0, 9, None, 0, None, None, None,
                                       None, None, None, None, None, 1, 1, 0, None, 0, None,
                                       None)
    assert rc == _lib.FFWD_ERR_VALIDATION and b"1..8 ranks" in lib.ffwd_last_error()


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU path")
def test_sequence_parallel_predictor_entries_validate_first():
    """ffwd_predict_mask / ffwd_ffn_layer_masked reject bad shapes and pointers before
    any launch (no device needed)."""
    lib = _lib.load_library()
    assert lib.ffwd_predict_mask_workspace_bytes(16, 4096, 256, 14336) > 16 * 14336 * 4
    dummy = ctypes.c_void_p(16)
    # ld_mask narrower than ceil(f / 32) words
    rc = lib.ffwd_predict_mask(dummy, 0, 1024, 512, 1, 6, dummy, dummy, dummy, 32, 1376, 688,
                               None, dummy, 10, dummy, 1 << 30, None)
    assert rc == _lib.FFWD_ERR_VALIDATION and b"ld_mask" in lib.ffwd_last_error()
    # blocks outside the tokens
    rc = lib.ffwd_predict_mask(dummy, 0, 1024, 512, 4, 6, dummy, dummy, dummy, 32, 1376, 688,
                               None, dummy, 43, dummy, 1 << 30, None)
    assert rc == _lib.FFWD_ERR_VALIDATION and b"outside" in lib.ffwd_last_error()
    # null mask
    rc = lib.ffwd_predict_mask(dummy, 0, 1024, 512, 1, 6, dummy, dummy, dummy, 32, 1376, 688,
                               None, None, 43, dummy, 1 << 30, None)
    assert rc == _lib.FFWD_ERR_VALIDATION
    # masked layer: bad rank, then predicted blocks without (wide enough) mask rows
    rc = lib.ffwd_ffn_layer_masked(dummy, 1024, 512, dummy, dummy, 688, 32, 1376, 688, 1, 1, 2,
                                   2, dummy, 43, dummy, None, None, dummy, 1 << 30, None)
    assert rc == _lib.FFWD_ERR_VALIDATION and b"rank" in lib.ffwd_last_error()
    rc = lib.ffwd_ffn_layer_masked(dummy, 1024, 512, dummy, dummy, 688, 32, 1376, 688, 1, 1, 0,
                                   2, dummy, 10, dummy, None, None, dummy, 1 << 30, None)
    assert rc == _lib.FFWD_ERR_VALIDATION and b"mask" in lib.ffwd_last_error()


def test_compute_path_fails_loudly_without_gpu():
    import paper_2602_00397_b200 as ff
    from oracle import ffwd_oracle as orc
    pred = orc.init_predictor(np.random.default_rng(0), 64, 200)
    x = np.ones((8, 64), np.float32)
    with pytest.raises(RuntimeError):
        ff.predictor_forward(ff.PredictorParams(**pred), x)
    with pytest.raises(RuntimeError):
        ff.topk_indices(np.ones(4, np.float32), 2)
    with pytest.raises(RuntimeError):
        _lib.require_device(0)
