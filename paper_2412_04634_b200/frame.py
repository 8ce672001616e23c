"""One frame of the online two-level renderer on the device: render with
θ_f, collect training paths, train → θ_{f+1} (experiment.py:149-185 of the
reference, the frame the 1080p < 10 ms target is quoted on).

Everything stays in device memory; the host touches the GPU twice per frame
(the record count after collection and the loss trace after training).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from .caches import default_train_count, train_frame
from .estimators import EstimatorConfig, render_and_collect, render_device


@dataclass
class FrameStats:
    queries: int
    records: int
    loss: float


def run_frame(scene, cache, config, seed, frame, spp=1, train_fraction=0.025, steps=4,
              batch=None, out=None):
    """Render frame `frame` and train the cache on it; returns
    ((img, img2, term) device sums, FrameStats)."""
    loss = math.nan
    nrec = 0
    if cache is None:
        img, img2, term, queries = render_device(scene, config, cache, seed, spp, frame, out=out)
    else:
        # render + training walks in one persistent trace launch
        img, img2, term, queries, rec = render_and_collect(
            scene, config, cache, seed, spp, frame,
            count=default_train_count(scene, train_fraction), out=out)
        nrec = len(rec)
        if nrec:
            trace = train_frame(cache, rec, steps=steps, batch=batch)
            loss = trace[-1]
    return (img, img2, term), FrameStats(int(queries.item()), nrec, loss)


def config3(nc=(16,)):
    """BASELINE config 3: two-level, nc=(16,) at the first cache vertex."""
    return EstimatorConfig(mode="two-level", nc=tuple(nc), max_cache_vertices=len(nc))
