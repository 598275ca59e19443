"""ctypes binding of ``libffwd_b200.so`` (the C-ABI in ``include/ffwd_b200.h``).

There is no CPU fallback: importing the compute entry points on a machine
without the built library or without an sm_100 GPU raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import UnsupportedError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFWD_LIB") or os.path.join(_HERE, "libffwd_b200.so")

FFWD_OK, FFWD_ERR_VALIDATION, FFWD_ERR_CUDA, FFWD_ERR_UNSUPPORTED = 0, 1, 2, 3

_c_int, _c_size, _vp = ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/ffwd_b200.h
SIGNATURES = {
    "ffwd_abi_version": (_c_int, []),
    "ffwd_last_error": (ctypes.c_char_p, []),
    "ffwd_device_check": (_c_int, [_c_int]),
    "ffwd_set_raster": (_c_int, [_c_int, _c_int]),
    "ffwd_set_serpentine": (_c_int, [_c_int]),
    "ffwd_set_spin_timeout_ms": (_c_int, [_c_int]),
    "ffwd_set_pdl": (_c_int, [_c_int]),
    "ffwd_predictor_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int, _c_int]),
    "ffwd_predictor_forward": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp,
                                        _vp, _c_int, _c_int, _vp, _vp, _c_size, _vp]),
    "ffwd_predictor_forward_block": (_c_int, [_vp, _c_int, _c_int, _c_int, _vp, _vp, _vp, _c_int,
                                              _c_int, _vp, _vp, _c_size, _vp]),
    "ffwd_predictor_logits": (_c_int, [_vp, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "ffwd_topk": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp,
                           _c_int, _vp, _vp]),
    "ffwd_predict_topk": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp,
                                   _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp,
                                   _c_int, _vp, _vp, _c_size, _vp]),
    "ffwd_sparse_ffn_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int, _c_int, _c_int]),
    "ffwd_sparse_ffn": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _vp, _c_int,
                                 _c_int, _vp, _c_int, _c_int, _vp, _vp, _c_size, _vp]),
    "ffwd_layer_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                                             _c_int, _c_int, _c_int]),
    "ffwd_ffn_layer": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _vp, _vp, _vp,
                                _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp,
                                _vp, _vp, _vp, _c_int, _vp, _c_size, _vp]),
    "ffwd_predict_mask_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int, _c_int]),
    "ffwd_predict_mask": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp,
                                   _c_int, _c_int, _c_int, _vp, _vp, _c_int, _vp, _c_size, _vp]),
    "ffwd_ffn_layer_masked": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int,
                                       _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp,
                                       _vp, _vp, _vp, _c_size, _vp]),
    "ffwd_ffn_layer2": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _vp, _vp, _vp,
                                 _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp,
                                 _vp, _vp, _vp, _c_int, _vp, _vp, _vp, _c_size, _vp]),
    "ffwd_hidden_scores_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int]),
    "ffwd_hidden_scores": (_c_int, [_vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _vp, _c_size,
                                    _vp]),
    "ffwd_column_norms": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp]),
    "ffwd_ffn_layer_mode_workspace_bytes": (_c_size, [_c_int] * 7),
    "ffwd_ffn_layer_mode": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int,
                                     _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _c_int, _vp,
                                     _c_size, _vp]),
    "ffwd_rmsnorm": (_c_int, [_vp, _vp, _c_int, _c_int, ctypes.c_double, _vp, _c_int, _vp, _vp,
                              _vp, _vp, _c_int, _c_int, _vp]),
    "ffwd_rmsnorm_ex": (_c_int, [_vp, _vp, _c_int, _c_int, ctypes.c_double, _vp, _c_int, _vp,
                                 _vp, _vp, _vp, _c_int, _c_int, _c_int, _vp]),
    "ffwd_rope": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp,
                           _vp, _c_int, _vp]),
    "ffwd_ckpt_last_error": (ctypes.c_char_p, []),
    "ffwd_ckpt_open": (_c_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "ffwd_ckpt_close": (None, [_vp]),
    "ffwd_ckpt_config": (_vp, [_vp, ctypes.POINTER(_c_size)]),
    "ffwd_ckpt_num_tensors": (_c_int, [_vp]),
    "ffwd_ckpt_tensor": (_c_int, [_vp, _c_int, ctypes.POINTER(ctypes.c_char_p),
                                  ctypes.POINTER(_c_int), ctypes.POINTER(ctypes.c_uint32),
                                  ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_uint64)]),
    "ffwd_allreduce_residual": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _c_int, _vp, _c_int, _c_int,
                                         ctypes.c_uint, _c_int, _vp]),
    "ffwd_ffn_layer_tp_overlap": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _vp,
                                           _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int,
                                           _c_int, _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp,
                                           _vp, _vp, _vp, ctypes.c_uint, ctypes.c_uint, _c_int,
                                           _vp, _c_size, _vp, _vp]),
    "ffwd_ipc_get_handle": (_c_int, [_vp, _vp, ctypes.POINTER(_c_size)]),
    "ffwd_ipc_open": (_c_int, [_vp, ctypes.POINTER(_vp)]),
    "ffwd_ipc_close": (_c_int, [_vp]),
    "ffwd_timing_enable": (_c_int, [_c_int]),
    "ffwd_timing_read": (_c_int, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_c_int),
                                  _c_int]),
    "ffwd_stage_name": (ctypes.c_char_p, [_c_int]),
}

_lib = None
_lock = threading.Lock()


def load_library() -> ctypes.CDLL:
    """Load the shared library and bind every exported symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                    "the hot path has no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status == FFWD_OK:
        return
    msg = load_library().ffwd_last_error().decode(errors="replace")
    if status == FFWD_ERR_VALIDATION:
        raise ValidationError(f"{what}: {msg}")
    if status == FFWD_ERR_UNSUPPORTED:
        raise UnsupportedError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA failure: {msg}")


_device_ok: dict[int, bool] = {}


def require_device(device_index: int) -> ctypes.CDLL:
    """The library, after checking that `device_index` is an sm_100 GPU."""
    lib = load_library()
    if device_index not in _device_ok:
        check(lib.ffwd_device_check(device_index), "ffwd_device_check")
        _device_ok[device_index] = True
    return lib
