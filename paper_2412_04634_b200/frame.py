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
from .records import collect_training_records


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


class ZeroWatch:
    """Cache.is_zero (caches.py:206-209) of a cache whose parameters change
    only through the pipeline's training: after each update the check runs on
    the device and lands in pinned memory asynchronously, so the next frame
    reads it without a host sync (None -> the caller checks synchronously)."""

    def __init__(self, cache):
        self.cache = cache
        self.host = torch.zeros((1,), dtype=torch.bool).pin_memory()
        self.ev = None
        self.value = None

    def after_update(self, stream):
        lo = int(self.cache.spec.w_off[-1])
        nz = torch.any(self.cache.theta[lo:] != 0)
        self.host.copy_(nz.reshape(1), non_blocking=True)
        self.ev = torch.cuda.Event()
        self.ev.record(stream)
        self.value = None

    def get(self):
        if self.value is None and self.ev is not None and self.ev.query():
            self.value = not bool(self.host[0])
        return self.value


class FramePipeline:
    """The same frame loop with rendering and training overlapped (SURVEY.md
    8(e) "render(f) || collect + train(f) on separate streams, double-buffered
    theta"):

      frame f:  theta_r <- theta_f                          (render stream)
                render(f) with theta_r  +  the training walks of frame f+1
                                         (one nirc_render_collect launch)
                train(f) on records(f) -> theta_{f+1}       (train stream)

    The walks never read theta, so collecting frame f+1's records during frame
    f's launch gives exactly the records run_frame collects at f+1; render(f)
    reads the snapshot of theta_f while train(f) updates theta.  Every frame's
    inputs are therefore run_frame's (the image of frame f, the records and
    the training steps are the same computations); only their overlap on the
    device differs.  Across an animation boundary (next frame's geometry
    differs) the next records are collected on their own at the next frame.
    """

    def __init__(self, scene, cache, config, seed, spp=1, train_fraction=0.025, steps=4,
                 batch=None):
        self.scene, self.cache, self.config = scene, cache, config
        self.seed, self.spp, self.steps, self.batch = seed, spp, steps, batch
        self.train_fraction = train_fraction
        self.s_render = torch.cuda.current_stream()
        self.s_train = torch.cuda.Stream()
        self.theta_r = torch.empty_like(cache.theta)
        self.pending = None  # (frame, Records or callable) for the next train
        self.zero = ZeroWatch(cache)

    def _count(self, scene):
        return default_train_count(scene, self.train_fraction)

    def step(self, frame, out=None):
        """Frame `frame`: returns ((img, img2, term), FrameStats)."""
        cache = self.cache
        scene = self.scene = self.scene.at_frame(frame)  # a new object only at a boundary
        cache.scene = scene
        # does an animation fire between this frame and the next?
        same_geometry = not any((a.frame <= frame + 1) != (a.frame <= frame)
                                for a in scene.desc.anims)
        if self.pending is not None and self.pending[0] == frame:
            rec = self.pending[1]
            rec = rec() if callable(rec) else rec
        else:
            rec = collect_training_records(scene, cache.seed, self._count(scene),
                                           cache.record_kind, frame)
        self.pending = None
        # theta_f snapshot for the render, after the previous training
        self.s_render.wait_stream(self.s_train)
        self.theta_r.copy_(cache.theta)
        snap = torch.cuda.Event()
        snap.record(self.s_render)
        zero = self.zero.get()
        if same_geometry:
            img, img2, term, queries, nxt_rec = render_and_collect(
                scene, self.config, cache, self.seed, self.spp, frame,
                count=self._count(scene), train_frame=frame + 1, out=out, theta=self.theta_r,
                defer=True, zero=zero)
            self.pending = (frame + 1, nxt_rec)
        else:
            img, img2, term, queries = render_device(scene, self.config, cache, self.seed,
                                                     self.spp, frame, out=out,
                                                     theta=self.theta_r, zero=zero)
        loss = math.nan
        self.train_events = None
        if len(rec):
            self.s_train.wait_event(snap)  # theta_f copied (the records are complete)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(self.s_train):
                t0.record(self.s_train)
                trace = train_frame(cache, rec, steps=self.steps, batch=self.batch)
                t1.record(self.s_train)
                self.zero.after_update(self.s_train)
            self.train_events = (t0, t1)
            loss = trace[-1]
        return (img, img2, term), FrameStats(int(queries.item()), len(rec), loss)
