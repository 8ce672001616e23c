"""Input encoding on the B200 (drop-in for pkg/src/nirclab/encoding.py).

``encode_batch`` and ``scatter_grid_grad`` run the sm_100a kernels in
csrc/neural.cu through the C ABI.  Slots, trilinear weights and the whole
encoded row are bit-identical to the reference's numpy path (f64
normalisation, f32 cell arithmetic, corner-ordered f32 accumulation, f64
SH rounded to f32).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib

P1 = 2654435761
P2 = 805459861
AUX_DIM = 7


def level_resolutions(levels, base_res, max_res):
    """Geometric ladder floor(base * b^l + 0.5), b = (max/base)^(1/(L-1))
    (encoding.py:29-35)."""
    if levels == 1:
        return np.array([base_res], np.int64)
    growth = np.exp(np.log(max_res / base_res) / (levels - 1))
    return np.floor(base_res * growth ** np.arange(levels) + 0.5).astype(np.int64)


def _c_spec(spec):
    return _lib.make_c_spec(spec)


def encode_batch(spec, theta, pos, normal, albedo, rough, dirs, dtype=None):
    """Returns (X, entries, weights) like encoding.py:111-157.

    X is (B, in_dim) float32, entries (B, levels, 8) int64 feature-table
    slots, weights (B, levels, 8) float32.
    """
    if dtype not in (None, np.float32, torch.float32):
        raise NotImplementedError("the device encoder produces float32 rows")
    host = _dev.is_host(pos)
    B = int(pos.shape[0])
    th = _dev.dev(theta, torch.float32)
    args = [_dev.dev(a, torch.float64) for a in (pos, normal, albedo, rough, dirs)]
    X = _dev.empty((B, spec.in_dim), torch.float32)
    ent = _dev.empty((B, spec.levels, 8), torch.int64)
    wts = _dev.empty((B, spec.levels, 8), torch.float32)
    lib = _lib.load()
    cs = _c_spec(spec)
    _lib.check(lib.nirc_encode(cs, _dev.ptr(th), *[_dev.ptr(a) for a in args], B,
                               _dev.ptr(X), _dev.ptr(ent), _dev.ptr(wts), _dev.stream()),
               "nirc_encode")
    return _dev.out(X, host), _dev.out(ent, host), _dev.out(wts, host)


def scatter_grid_grad(spec, grad_theta, entries, weights, dX):
    """grad[slot*F + f] += w * dX[:, l*F + f] (encoding.py:160-167), in place."""
    host = _dev.is_host(grad_theta)
    g = _dev.dev(grad_theta, torch.float32)
    e = _dev.dev(entries, torch.int64)
    w = _dev.dev(weights, torch.float32)
    d = _dev.dev(dX, torch.float32)
    n = int(e.shape[0])
    lib = _lib.load()
    _lib.check(lib.nirc_scatter_grid_grad(_c_spec(spec), _dev.ptr(g), _dev.ptr(e), _dev.ptr(w),
                                          _dev.ptr(d), n, int(d.shape[1]), _dev.stream()),
               "nirc_scatter_grid_grad")
    if host:
        grad_theta[...] = g.cpu().numpy()
    elif g.data_ptr() != grad_theta.data_ptr():
        grad_theta.copy_(g)
    return grad_theta
