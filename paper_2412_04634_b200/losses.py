"""Training losses on the device (drop-in for pkg/src/nirclab/losses.py).

Each returns (float mean loss, dL/dY).  The kernels follow the reference's
numpy promotions: f32 prediction, f64 target/pdf, the relative-L2
denominator f32(y*y) + f32(eps), the gradient computed in f64.  As in
train_frame (caches.py:349) the returned gradient is float32.
"""

from __future__ import annotations

import torch

from . import _dev, _lib
from .errors import DivergenceError, InvalidSampleError

_KIND = {"l2": 0, "relative_l2": 1, "variance": 2, "bce": 3}


def _run_f64(kind, prediction, target, pdf, eps=0.01, running_mean=None, frozen=None):
    """float64 predictions: every operation in f64, gradient float64 (the
    reference's numpy promotions for an f64 prediction)."""
    host = _dev.is_host(prediction)
    y = _dev.dev(prediction, torch.float64)
    n = int(y.shape[0])
    t = _dev.dev(target, torch.float64)
    p = _dev.dev(pdf, torch.float64) if pdf is not None else _dev.zeros((n,), torch.float64)
    rm = _dev.dev(running_mean, torch.float64) if running_mean is not None else None
    den = _dev.dev(frozen, torch.float64) if frozen is not None else None
    dY = _dev.empty((n, 3), torch.float64)
    loss = _dev.zeros((1,), torch.float64)
    flags = _dev.zeros((1,), torch.int32)
    lib = _lib.load()
    _lib.check(lib.nirc_loss_f64(_KIND[kind], _dev.ptr(y), _dev.ptr(t), _dev.ptr(p),
                                 _dev.ptr(rm), _dev.ptr(den), float(eps), n, _dev.ptr(dY),
                                 _dev.ptr(loss), _dev.ptr(flags), _dev.stream()), "nirc_loss_f64")
    if int(flags.item()) & 1:
        raise InvalidSampleError("sample pdf must be positive")
    return float(loss.item()), _dev.out(dY, host)


def _run(kind, prediction, target, pdf, eps=0.01, running_mean=None):
    if _dev.is_f64(prediction):
        return _run_f64(kind, prediction, target, pdf, eps, running_mean)
    host = _dev.is_host(prediction)
    y = _dev.dev(prediction, torch.float32)
    n = int(y.shape[0])
    t = _dev.dev(target, torch.float64)
    p = _dev.dev(pdf, torch.float64) if pdf is not None else _dev.zeros((n,), torch.float64)
    rm = _dev.dev(running_mean, torch.float64) if running_mean is not None else None
    dY = _dev.empty((n, 3), torch.float32)
    loss = _dev.zeros((1,), torch.float64)
    flags = _dev.zeros((1,), torch.int32)
    scratch = _dev.empty(((n + 255) // 256 + 2) * 3, torch.float64)
    lib = _lib.load()
    _lib.check(lib.nirc_loss(_KIND[kind], _dev.ptr(y), _dev.ptr(t), _dev.ptr(p), _dev.ptr(rm),
                             float(eps), n, _dev.ptr(dY), _dev.ptr(loss), _dev.ptr(flags),
                             _dev.ptr(scratch), _dev.stream()), "nirc_loss")
    f = int(flags.item())
    if f & 1:
        raise InvalidSampleError("sample pdf must be positive")
    return float(loss.item()), _dev.out(dY, host)


def loss_l2(prediction, target, pdf):
    return _run("l2", prediction, target, pdf)


def loss_relative_l2(prediction, target, pdf, eps=0.01, frozen_denom=None):
    """frozen_denom (the finite-difference helper's captured y*y + eps) is
    honoured for float64 predictions; the f32 device loss freezes it itself."""
    if frozen_denom is not None:
        if not _dev.is_f64(prediction):
            raise NotImplementedError("frozen denominators are supported in the float64 "
                                      "shadow mode")
        return _run_f64("relative_l2", prediction, target, pdf, eps=eps, frozen=frozen_denom)
    return _run("relative_l2", prediction, target, pdf, eps=eps)


def loss_variance(prediction, target, pdf, running_mean):
    return _run("variance", prediction, target, pdf, running_mean=running_mean)


def loss_bce(prediction, target):
    return _run("bce", prediction, target, None)


def relative_l2_denom(prediction, eps=0.01):
    return prediction * prediction + eps


__all__ = ["loss_l2", "loss_relative_l2", "loss_variance", "loss_bce", "relative_l2_denom",
           "DivergenceError"]
