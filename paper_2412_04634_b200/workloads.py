"""Synthetic workloads of BASELINE.json's configs (host-generated, uploaded).

``measure_queries`` is config 2's query recipe: columns
drawn from the P_MEASURE splitmix64 streams 0..4 -- pos in [0,1)^3, unit
normals and directions from normalised ``normal_array`` triples, albedo
U[0,1)^3, roughness U[0,1).
"""

from __future__ import annotations

import numpy as np
import torch

from . import rng


def measure_queries(n, seed=0):
    P = rng.P_MEASURE
    pos = rng.uniform_array(seed, P, 0, 3 * n).reshape(n, 3)
    nrm = rng.normal_array(seed, P, 1, 3 * n).reshape(n, 3)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    alb = rng.uniform_array(seed, P, 2, 3 * n).reshape(n, 3)
    rough = rng.uniform_array(seed, P, 3, n)
    dirs = rng.normal_array(seed, P, 4, 3 * n).reshape(n, 3)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return pos, nrm, alb, rough, dirs


def measure_queries_device(n, seed=0):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in measure_queries(n, seed)]
