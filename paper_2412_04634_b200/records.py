"""Training-record collection on the device (collect_training_records,
pkg/src/nirclab/caches.py:87-131 over kernels.py:85-311).

Records stay in device memory (f64, the reference's row order: path-major,
vertex-minor); the record count is read back once per call.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _dev, _lib
from .caches import RECORD_KINDS, Records
from .errors import ConfigError

_KIND = {"nirc": 0, "nirc_full": 1, "nrc": 2, "nvc": 3, "nirc_env": 4}


class _CollectWs:
    buf = None

    @classmethod
    def get(cls, nbytes):
        if cls.buf is None or cls.buf.numel() < nbytes:
            cls.buf = _dev.empty((max(int(nbytes), 256),), torch.uint8)
        return cls.buf


def _check_kind(scene, kind):
    if kind not in RECORD_KINDS:
        raise ConfigError(f"unknown record kind '{kind}'")
    if kind in ("nvc", "nirc_env") and scene.pack.env_kind == 0:
        raise ConfigError(f"record kind '{kind}' needs an environment light")
    if kind not in _KIND:
        raise NotImplementedError(f"record kind '{kind}' is outside the NIRC hot path")


def record_buffers(count):
    """Output columns for `count` training paths (<= 63 records each)."""
    cap = int(count) * 63
    out = {k: _dev.empty((cap, 3), torch.float64) for k in ("pos", "ns", "alb", "dirs", "target")}
    out["rough"] = _dev.empty((cap,), torch.float64)
    out["pdf"] = _dev.empty((cap,), torch.float64)
    ro = _lib.NircRecordsOut()
    for k, t in out.items():
        setattr(ro, k, t.data_ptr())
    ro.cap = cap
    return out, ro


def collect_training_records(scene, seed, count, kind="nirc", frame=0):
    _check_kind(scene, kind)
    count = int(count)
    out, ro = record_buffers(count)
    n_out = _dev.zeros((1,), torch.int64)
    lib = _lib.load()
    ws = _CollectWs.get(lib.nirc_collect_workspace_bytes(count))
    ds = scene.device()
    _lib.check(lib.nirc_collect(ds.ptr(), _dev.ptr(ds.cam), int(seed), int(frame), count,
                                _KIND[kind], C.byref(ro), _dev.ptr(n_out), _dev.ptr(ws),
                                int(ws.numel()), _dev.stream()), "nirc_collect")
    n = int(n_out.item())
    return Records(kind=kind, frame=frame, n=n, **{k: v[:n] for k, v in out.items()})
