"""Device plumbing: torch supplies device memory and streams; libs2v computes.

Every rank (thread in run_workers, or process under torchrun) binds one CUDA
device.  Raises immediately when no CUDA device is present: the package has
no CPU compute path.
"""
from __future__ import annotations

import threading

import numpy as np
import torch

_tls = threading.local()

NP_TO_TORCH = {
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.uint8): torch.uint8,
}


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2105_08764_b200 needs a CUDA device (sm_100a); there is no CPU fallback")


def bind_device(device: int | None = None) -> torch.device:
    """Bind the calling thread to a CUDA device (default: the current one)."""
    require_cuda()
    if device is None:
        device = getattr(_tls, "device", None)
        if device is None:
            device = torch.cuda.current_device()
    torch.cuda.set_device(device)
    from . import _lib
    _lib.call("s2v_set_device", int(device))
    _tls.device = int(device)
    return torch.device("cuda", int(device))


def current_device() -> torch.device:
    dev = getattr(_tls, "device", None)
    if dev is None:
        return bind_device()
    torch.cuda.set_device(dev)
    return torch.device("cuda", dev)


def stream_ptr() -> int:
    """Raw cudaStream_t of the current torch stream on this thread's device."""
    return torch.cuda.current_stream(current_device()).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def to_device(arr: np.ndarray, device=None, pinned: bool = False) -> torch.Tensor:
    """Host array -> new device tensor.  pinned: stage through page-locked
    memory and copy asynchronously on the current stream (ordered before any
    later kernel on that stream)."""
    arr = np.ascontiguousarray(arr)
    t = torch.from_numpy(arr)
    if pinned:
        return t.pin_memory().to(device or current_device(), non_blocking=True)
    return t.to(device or current_device(), non_blocking=False)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()
