"""Minimal PFM reader/writer (the reference's artifact format,
pkg/src/nirclab/pfm.py), used for lat-long environments and images."""

from __future__ import annotations

import numpy as np

from .errors import ConfigError


def write_pfm(path, img):
    a = np.asarray(img, np.float32)
    if a.ndim == 2:
        a = np.repeat(a[:, :, None], 3, axis=2)
    h, w = a.shape[:2]
    with open(path, "wb") as fh:
        fh.write(f"PF\n{w} {h}\n-1.0\n".encode())
        fh.write(np.ascontiguousarray(a[::-1]).astype("<f4").tobytes())


def read_pfm(path):
    with open(path, "rb") as fh:
        head = fh.readline().strip()
        if head not in (b"PF", b"Pf"):
            raise ConfigError(f"not a PFM file: {path}")
        w, h = (int(v) for v in fh.readline().split())
        scale = float(fh.readline())
        ch = 3 if head == b"PF" else 1
        data = np.frombuffer(fh.read(), "<f4" if scale < 0 else ">f4")
    if data.size != w * h * ch:
        raise ConfigError(f"truncated PFM file: {path}")
    return data.reshape(h, w, ch)[::-1].astype(np.float32)
