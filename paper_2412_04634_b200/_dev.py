"""Device-memory plumbing: torch owns every buffer, the C ABI sees pointers.

Public functions of the drop-in API accept numpy arrays (the reference's
types) or torch tensors.  numpy inputs are uploaded and the results come
back as numpy; CUDA tensors stay on the device end to end.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("the NIRC B200 path needs a CUDA device (no CPU fallback)")


def is_host(x):
    return not (isinstance(x, torch.Tensor) and x.is_cuda)


def dev(x, dtype, shape=None):
    """Contiguous CUDA tensor of the given dtype (copying only if needed)."""
    require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.cuda()
        if t.dtype != dtype:
            t = t.to(dtype)
    else:
        a = np.ascontiguousarray(np.asarray(x), dtype=_np_dtype(dtype))
        t = torch.from_numpy(a).cuda(non_blocking=False)
    t = t.contiguous()
    if shape is not None:
        t = t.reshape(shape)
    return t


def _np_dtype(dtype):
    return {torch.float32: np.float32, torch.float64: np.float64,
            torch.int64: np.int64, torch.int32: np.int32, torch.uint8: np.uint8,
            torch.bool: np.bool_}[dtype]


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def out(t, host):
    """Return t as numpy when the caller passed host arrays."""
    if host:
        return t.cpu().numpy()
    return t


def empty(shape, dtype):
    require_cuda()
    return torch.empty(shape, dtype=dtype, device="cuda")


def zeros(shape, dtype):
    require_cuda()
    return torch.zeros(shape, dtype=dtype, device="cuda")


def is_f64(x):
    """True for float64 arrays / tensors (the reference's 64-bit shadow mode)."""
    if isinstance(x, torch.Tensor):
        return x.dtype == torch.float64
    return getattr(x, "dtype", None) == np.float64
