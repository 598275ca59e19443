"""Device plumbing: host<->device conversion, stream handles, workspaces.

PyTorch is used only for device memory and streams; all arithmetic of the
hot path happens in libffwd_b200.so.
"""

from __future__ import annotations

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


_ws: dict[int, torch.Tensor] = {}


def workspace(device: torch.device, nbytes: int) -> torch.Tensor:
    """A per-device scratch buffer that only grows (stream-ordered reuse)."""
    idx = device.index if device.index is not None else 0
    buf = _ws.get(idx)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _ws[idx] = buf
    return buf


def is_host(a) -> bool:
    return not (isinstance(a, torch.Tensor) and a.is_cuda)


def to_host_f32(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float32).numpy()
