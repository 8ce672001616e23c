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


def is_default_layout(spec):
    """The 12 x 2 hash + 4-band SH input the fused kernels are built for."""
    return (int(spec.levels) == 12 and int(spec.feats) == 2 and int(spec.bands) == 4
            and int(spec.in_dim) == 47)


def _c_spec(spec):
    return _lib.make_c_spec(spec)


def encode_batch(spec, theta, pos, normal, albedo, rough, dirs, dtype=None):
    """Returns (X, entries, weights) like encoding.py:111-157.

    X is (B, in_dim) in ``dtype`` (default: theta's dtype, as the
    reference), entries (B, levels, 8) int64 feature-table slots, weights
    (B, levels, 8) float32.  float64 = the reference's shadow mode: the
    features accumulate in f64, SH and aux are not rounded to f32."""
    if dtype is None:
        dtype = np.float64 if _dev.is_f64(theta) else np.float32
    if dtype in (np.float64, torch.float64):
        return _encode_batch_f64(spec, theta, pos, normal, albedo, rough, dirs)
    if dtype not in (np.float32, torch.float32):
        raise NotImplementedError(f"encode_batch dtype {dtype}")
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


def _encode_batch_f64(spec, theta, pos, normal, albedo, rough, dirs):
    host = _dev.is_host(pos)
    B = int(pos.shape[0])
    th = _dev.dev(theta, torch.float64)
    args = [_dev.dev(a, torch.float64) for a in (pos, normal, albedo, rough, dirs)]
    X = _dev.empty((B, spec.in_dim), torch.float64)
    ent = _dev.empty((B, spec.levels, 8), torch.int64)
    wts = _dev.empty((B, spec.levels, 8), torch.float32)
    lib = _lib.load()
    _lib.check(lib.nirc_encode_f64(_c_spec(spec), _dev.ptr(th), *[_dev.ptr(a) for a in args], B,
                                   _dev.ptr(X), _dev.ptr(ent), _dev.ptr(wts), _dev.stream()),
               "nirc_encode_f64")
    return _dev.out(X, host), _dev.out(ent, host), _dev.out(wts, host)


def scatter_grid_grad(spec, grad_theta, entries, weights, dX):
    """grad[slot*F + f] += w * dX[:, l*F + f] (encoding.py:160-167), in place,
    in np.add.at's order (bit-identical given identical inputs)."""
    if _dev.is_f64(grad_theta):
        host = _dev.is_host(grad_theta)
        g = _dev.dev(grad_theta, torch.float64)
        e = _dev.dev(entries, torch.int64)
        w = _dev.dev(weights, torch.float32)
        d = _dev.dev(dX, torch.float64)
        lib = _lib.load()
        _lib.check(lib.nirc_scatter_grid_grad_f64(_c_spec(spec), _dev.ptr(g), _dev.ptr(e),
                                                  _dev.ptr(w), _dev.ptr(d), int(e.shape[0]),
                                                  int(d.shape[1]), _dev.stream()),
                   "nirc_scatter_grid_grad_f64")
        if host:
            grad_theta[...] = g.cpu().numpy()
        elif g.data_ptr() != grad_theta.data_ptr():
            grad_theta.copy_(g)
        return grad_theta
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


# ---- scalar per-surface API (encoding.py:45-108, :170-192) ----------------
_ZERO_GRIDS = {}


def _encode_rows(spec, theta, pos, normal, albedo, rough, dirs):
    """Device encoder on a handful of rows -> float32 numpy (n, in_dim)."""
    f = lambda a, w: np.asarray(a, np.float64).reshape(-1, w)  # noqa: E731
    X, _, _ = encode_batch(spec, theta, f(pos, 3), f(normal, 3), f(albedo, 3),
                           np.asarray(rough, np.float64).reshape(-1), f(dirs, 3))
    return X


def encode_surface_into(spec, theta, px, py, pz, nx, ny, nz, ar, ag, ab, rough, xin):
    """Hash-grid + aux blocks of one surface into xin (encoding.py:45-101);
    the SH block of xin is left as it is.  Runs the device encoder."""
    X = _encode_rows(spec, theta, (px, py, pz), (nx, ny, nz), (ar, ag, ab), rough,
                     (0.0, 0.0, 1.0))[0]
    g = spec.levels * spec.feats
    a0 = g + spec.bands * spec.bands
    xin[:g] = X[:g]
    xin[a0:a0 + AUX_DIM] = X[a0:a0 + AUX_DIM]
    return xin


def encode_dir_into(spec, dx, dy, dz, xin):
    """SH block of one direction into xin (encoding.py:104-108), evaluated
    by the device encoder (f64 recurrences rounded to f32)."""
    key = int(spec.grid_len), int(spec.theta_len)
    th = _ZERO_GRIDS.get(key)
    if th is None:
        th = _dev.zeros((int(spec.theta_len),), torch.float32)
        _ZERO_GRIDS[key] = th
    X = _encode_rows(spec, th, (0.0, 0.0, 0.0), (0.0, 0.0, 1.0), (0.0, 0.0, 0.0), 0.0,
                     (dx, dy, dz))[0]
    g = spec.levels * spec.feats
    s = spec.bands * spec.bands
    xin[g:g + s] = X[g:g + s]
    return xin


def encode(surface, wi, grids, bands=None):
    """One full encoded input (position, direction, aux) as a float64 vector
    (encoding.py:170-192).  surface = (position, normal, albedo, roughness);
    grids has .spec and .theta (a cache or a bare net)."""
    from .errors import ConfigError

    spec, theta = grids.spec, grids.theta
    if bands is not None and bands != spec.bands:
        raise ConfigError(f"encode bands {bands} does not match network bands {spec.bands}")
    pos, normal, albedo, rough = surface
    return _encode_rows(spec, theta, pos, normal, albedo, rough, wi)[0].astype(np.float64)
