"""Device plumbing: host<->device conversion, stream handles, workspaces.

PyTorch is used only for device memory and streams; all arithmetic of the
hot path happens in libffwd_b200.so.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib


def device_of(*objs) -> torch.device:
    for o in objs:
        if isinstance(o, torch.Tensor) and o.is_cuda:
            return o.device
    if not torch.cuda.is_available():
        raise RuntimeError("the FastForward hot path needs a CUDA (sm_100a) device; "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(a, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA tensor of `dtype` (bf16 rounding is RNE)."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32)))
    return t.to(device=device, dtype=dtype, non_blocking=True).contiguous()


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def lib_for(device: torch.device):
    return _lib.require_device(device.index if device.index is not None else 0)


_ws: dict[tuple[int, int], torch.Tensor] = {}
_ws_lock = threading.Lock()


def workspace(device: torch.device, nbytes: int) -> torch.Tensor:
    """Scratch for the current stream of `device`, grow-only, one buffer per stream.

    Calls on the same stream are ordered, so they can share one buffer; two streams
    never do.  A grown buffer replaces the old one, whose memory the caching allocator
    hands back only to work on the same stream (its allocation stream), after the work
    already queued there, so in-flight kernels never see it reused."""
    idx = device.index if device.index is not None else 0
    key = (idx, torch.cuda.current_stream(device).cuda_stream)
    with _ws_lock:
        buf = _ws.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            _ws[key] = buf
        return buf


def fingerprint(*arrays) -> tuple:
    """Cheap identity + content key of host / device arrays, for caches of derived device
    data (packed weights): the buffer address, shape and dtype, plus torch's in-place
    version counter for tensors or a strided content sample for numpy arrays (an in-place
    edit of a numpy array that misses every sampled element is not seen: call
    ``layer.invalidate_packed`` after editing weights in place)."""
    key = []
    for a in arrays:
        if a is None:
            key.append(None)
        elif isinstance(a, torch.Tensor):
            key.append(("t", a.data_ptr(), tuple(a.shape), str(a.dtype), a._version))
        else:
            arr = np.asarray(a)
            flat = arr.reshape(-1)
            step = max(1, flat.size // 4096)
            sample = np.ascontiguousarray(flat[::step])
            key.append(("n", arr.__array_interface__["data"][0], arr.shape, arr.dtype.str,
                        hash(sample.tobytes())))
    return tuple(key)


def cached_on(obj, slot: str, key, build):
    """`build()` memoised on `obj` itself (its ``__dict__``) under `slot`, valid while `key`
    (a fingerprint) is unchanged.  The cache lives and dies with the object, so no global
    table keyed by ``id()`` can go stale."""
    store = getattr(obj, "__dict__", None)
    if store is None:
        return build()
    hit = store.get(slot)
    if hit is not None and hit[0] == key:
        return hit[1]
    val = build()
    store[slot] = (key, val)
    return val


def is_host(a) -> bool:
    return not (isinstance(a, torch.Tensor) and a.is_cuda)


def to_host_f32(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float32).numpy()
