"""Dense Adam on the device (drop-in for pkg/src/nirclab/adam.py).

m, v, t and the skip counter live in device memory; ``adam_step`` runs the
reference's exact f32 sequence (bit-identical given identical gradients)
and skips the whole step, without advancing t, on any non-finite gradient.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib


class AdamState:
    def __init__(self, theta, lr=0.01, beta1=0.9, beta2=0.99, eps=1e-8):
        n = int(theta.shape[0]) if hasattr(theta, "shape") else len(theta)
        dt = torch.float64 if _dev.is_f64(theta) else torch.float32  # zeros_like(theta)
        self.m = _dev.zeros((n,), dt)
        self.v = _dev.zeros((n,), dt)
        self._t = _dev.zeros((1,), torch.int64)
        self._skipped = _dev.zeros((1,), torch.int64)
        self._scratch = _dev.zeros((4,), torch.int32)
        self.lr = lr
        self.beta1 = beta1
        self.beta2 = beta2
        self.eps = eps

    @property
    def t(self):
        return int(self._t.item())

    @t.setter
    def t(self, value):
        self._t.fill_(int(value))

    @property
    def skipped(self):
        return int(self._skipped.item())

    @skipped.setter
    def skipped(self, value):
        self._skipped.fill_(int(value))


def _adam_step_f64(state, theta, grad):
    host = _dev.is_host(theta)
    th = _dev.dev(theta, torch.float64)
    g = _dev.dev(grad, torch.float64)
    before = state.skipped
    lib = _lib.load()
    _lib.check(lib.nirc_adam_step_f64(_dev.ptr(th), _dev.ptr(state.m), _dev.ptr(state.v),
                                      _dev.ptr(g), int(th.shape[0]), _dev.ptr(state._t),
                                      _dev.ptr(state._skipped), float(state.lr),
                                      float(state.beta1), float(state.beta2), float(state.eps),
                                      _dev.ptr(state._scratch), _dev.stream()),
               "nirc_adam_step_f64")
    if host:
        theta[...] = th.cpu().numpy()
    elif th.data_ptr() != theta.data_ptr():
        theta.copy_(th)
    return state.skipped == before


def adam_step(state, theta, grad):
    """One in-place update; returns False when the step was skipped.  A
    float64 theta (the reference's shadow mode) updates f64 state."""
    if _dev.is_f64(theta):
        return _adam_step_f64(state, theta, grad)
    host = _dev.is_host(theta)
    th = _dev.dev(theta, torch.float32)
    g = _dev.dev(grad, torch.float32)
    before = state.skipped
    lib = _lib.load()
    _lib.check(lib.nirc_adam_step(_dev.ptr(th), _dev.ptr(state.m), _dev.ptr(state.v),
                                  _dev.ptr(g), int(th.shape[0]), _dev.ptr(state._t),
                                  _dev.ptr(state._skipped), float(state.lr),
                                  float(state.beta1), float(state.beta2), float(state.eps),
                                  None, _dev.ptr(state._scratch), _dev.stream()),
               "nirc_adam_step")
    if host:
        theta[...] = th.cpu().numpy().astype(np.asarray(theta).dtype)
    elif th.data_ptr() != theta.data_ptr():
        theta.copy_(th)
    return state.skipped == before
