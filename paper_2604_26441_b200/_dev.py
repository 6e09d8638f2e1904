"""Device plumbing: torch is used only for CUDA allocation, streams and
host<->device copies; all arithmetic happens in libsg_b200.so kernels."""

from __future__ import annotations

import numpy as np

try:
    import torch
except ImportError as exc:  # pragma: no cover - torch is part of the image
    raise ImportError("paper_2604_26441_b200 needs PyTorch for device memory") from exc

from . import _native

_F64 = torch.float64
_F32 = torch.float32
_PINNED_MIN = 1 << 20  # results / inputs this large go through pinned staging


def device():
    if not torch.cuda.is_available():
        raise _native.NativeError("no CUDA device: the sm_100a solver has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    """Raw cudaStream_t of torch's current stream (the launch stream)."""
    return C_void(torch.cuda.current_stream().cuda_stream)


def C_void(v):
    import ctypes
    return ctypes.c_void_p(int(v))


def ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def is_device_tensor(x):
    return isinstance(x, torch.Tensor) and x.is_cuda


def as_device(x, dtype=np.float64, n=None):
    """(contiguous CUDA tensor of dtype, was_host) for numpy / torch input."""
    tdt = _F64 if np.dtype(dtype) == np.float64 else _F32
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if not t.is_cuda:
            t = t.to(device())
        if t.dtype != tdt:
            t = t.to(tdt)
        t = t.contiguous().reshape(-1)
        host = False
    else:
        dev = device()  # raises NativeError first on a box without a GPU
        a = np.ascontiguousarray(np.asarray(x), dtype=dtype).reshape(-1)
        src = torch.from_numpy(a)
        if a.nbytes >= _PINNED_MIN:
            # staged through page-locked memory (torch's caching host allocator,
            # which keeps the buffer until the async copy completes): a
            # multithreaded host memcpy + a full-rate DMA instead of the
            # driver's pageable path (24.5 MB: 1.22 -> 0.71 ms on the B200 box)
            pin = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
            pin.copy_(src)
            t = pin.to(dev, non_blocking=True)
        else:
            t = src.to(dev, non_blocking=False)
        host = True
    if n is not None and t.numel() != n:
        raise ValueError(f"expected free vector of length {n}")
    return t, host


def empty(n, dtype=np.float64):
    tdt = _F64 if np.dtype(dtype) == np.float64 else _F32
    return torch.empty(int(n), dtype=tdt, device=device())


def zeros(n, dtype=np.float64):
    tdt = _F64 if np.dtype(dtype) == np.float64 else _F32
    return torch.zeros(int(n), dtype=tdt, device=device())



def back(t, host):
    """Return numpy (for host callers) or the device tensor.  Large results are
    copied into page-locked memory (torch's caching host allocator) so the D2H
    runs at the full link rate; the numpy array keeps that buffer alive."""
    if host:
        if t.numel() * t.element_size() >= _PINNED_MIN:
            out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            out.copy_(t)
            return out.numpy()
        return t.cpu().numpy()
    return t
