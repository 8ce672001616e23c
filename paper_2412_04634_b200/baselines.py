"""Batch consumers of fused inference from the control-variate baselines
(SURVEY.md 8(f) item 3): the per-pixel integrand sampler the reference's
`residual_variance_report` streams (baselines.py:426-431 over
kernels.py:342-421) and the cache's prediction at every live draw
(`_nirc_grid_eval`, baselines.py:434-446).

Both run on the device: `integrand_round` launches one thread per (pixel,
draw) through `nirc_integrand_samples`; `nirc_grid_eval` gathers the live
draws' surface rows and directions and calls the fused encode + MLP kernel
(`nirc_full_forward`).  The reference-signature wrappers `_integrand_round`
and `_nirc_grid_eval` take and return numpy like the reference's.

The analytic SH / vMF control variates themselves (baselines.py:46-345) are
host-side fitting code outside the hot path.
"""

import numpy as np
import torch

from . import _dev, _lib
from .mlp import full_forward

_KEYS = ("dir", "f", "frc", "pdf", "valid", "spos", "sns", "salb", "srough")


def integrand_buffers(scene, per_round):
    """Zeroed device buffers of one integrand round (the reference's `out`
    dict, baselines.py:471-476): dir / f / frc (P, K, 3), pdf (P, K), valid
    (P,) u8, spos / sns / salb (P, 3), srough (P,)."""
    w, h = int(scene.camera[14]), int(scene.camera[15])
    p_, k_ = w * h, int(per_round)
    f64 = torch.float64
    return dict(dir=_dev.zeros((p_, k_, 3), f64), f=_dev.zeros((p_, k_, 3), f64),
                frc=_dev.zeros((p_, k_, 3), f64), pdf=_dev.zeros((p_, k_), f64),
                valid=_dev.zeros((p_,), torch.uint8), spos=_dev.zeros((p_, 3), f64),
                sns=_dev.zeros((p_, 3), f64), salb=_dev.zeros((p_, 3), f64),
                srough=_dev.zeros((p_,), f64))


def integrand_round(scene, seed, frame, per_round, out):
    """integrand_samples_kernel (kernels.py:342-421) into the device dict
    `out` (from `integrand_buffers`); entries the reference leaves untouched
    keep their previous values."""
    if int(per_round) <= 0:
        raise ValueError("per_round must be positive")
    ds = scene.device()
    lib = _lib.load()
    _lib.check(lib.nirc_integrand_samples(
        ds.ptr(), _dev.ptr(ds.cam), int(seed), int(frame), int(per_round),
        *[_dev.ptr(out[k]) for k in _KEYS], _dev.stream()), "nirc_integrand_samples")
    return out


def _integrand_round(scene, seed, frame, per_round, scratch, out):
    """baselines.py:426-431 over numpy `out` arrays (scratch is the
    reference's host walk scratch; the device walks carry their own)."""
    dev = {k: _dev.dev(np.asarray(out[k]), torch.uint8 if k == "valid" else torch.float64)
           for k in _KEYS}
    integrand_round(scene, seed, frame, per_round, dev)
    for k in _KEYS:
        out[k][...] = dev[k].cpu().numpy()


def nirc_grid_eval(cache, out, live):
    """Cache predictions times brdf * cos at every live draw, (P, K, 3) f64,
    on the device (baselines.py:434-446): one fused full_forward over the
    live draws' surface rows and directions."""
    p_, k_ = int(out["dir"].shape[0]), int(out["dir"].shape[1])
    live = live.reshape(-1)
    idx = torch.nonzero(live).reshape(-1)
    g = _dev.zeros((p_ * k_, 3), torch.float64)
    if idx.numel():
        pix = idx // k_
        pred = full_forward(cache.spec, cache.theta, out["spos"][pix], out["sns"][pix],
                            out["salb"][pix], out["srough"][pix],
                            out["dir"].reshape(-1, 3)[idx])
        g[idx] = pred.to(torch.float64)
    return g.reshape(p_, k_, 3) * out["frc"]


def _nirc_grid_eval(cache, out, live):
    """baselines.py:434-446 with the reference's numpy types."""
    dev = {k: _dev.dev(np.asarray(out[k]), torch.float64) for k in
           ("dir", "frc", "spos", "sns", "salb", "srough")}
    return nirc_grid_eval(cache, dev, _dev.dev(np.asarray(live), torch.bool)).cpu().numpy()
