"""Rendering estimators on the B200 (drop-in for pkg/src/nirclab/estimators.py:
render, render_two_level, render_biased, EstimatorConfig, RenderResult).

``render`` runs the device frame pipeline (C-ABI ``nirc_render``): fp64 path
tracing with deferred cache vertices, the fused tcgen05 inference + MLMC
combine, and per-pixel accumulation.  The biased early-stop modes
(biased-nirc-bth / -sph, biased-nrc-sph, kernels.py:609-720) run through the
same kernels: their stop vertex is a deferred cache vertex with nbias
directions (or one NRC query at wo).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .errors import ConfigError

T_FAR = 1.0e30  # geometry.py:16

MODES = {"pt": 0, "two-level": 1, "biased-nirc-bth": 2, "biased-nirc-sph": 3,
         "biased-nrc-sph": 4}
MAX_DIRS = 28  # OFF_CACHE leaves room for 28 direction pairs per vertex

# network arithmetic of the fused inference (include/nirc_b200.h)
PRECISION_TF32X3, PRECISION_FP32, PRECISION_F16X2 = 0, 1, 2
DEFAULT_PRECISION = PRECISION_F16X2


@dataclass
class EstimatorConfig:
    """Render-mode knobs (estimators.py:49-84)."""

    mode: str = "pt"
    nc: tuple = (15, 5, 5)
    nbias: int = 5
    nr: int = 1
    max_cache_vertices: int = 3
    sph_c: float = 0.01
    rr: float = 0.1
    roughness_cutoff: float = 0.0625

    def __post_init__(self):
        if self.mode not in MODES:
            raise ConfigError(f"unknown estimator mode '{self.mode}'")
        if len(self.nc) < self.max_cache_vertices:
            raise ConfigError("nc must cover max_cache_vertices entries")
        for v in self.nc:
            if not 0 <= int(v) <= MAX_DIRS:
                raise ConfigError(f"nc entry {v} outside 0..{MAX_DIRS}")
        if not 1 <= self.nbias <= MAX_DIRS:
            raise ConfigError(f"nbias {self.nbias} outside 1..{MAX_DIRS}")
        if self.nr != 1:
            raise ConfigError("the walk carries exactly one residual sample per cache vertex")
        if not 0.0 <= self.rr < 1.0:
            raise ConfigError(f"roulette probability {self.rr} not in [0,1)")
        if self.sph_c <= 0.0:
            raise ConfigError("spread threshold must be positive")


@dataclass
class RenderResult:
    image: np.ndarray
    sample_var: np.ndarray
    path_length: np.ndarray
    spp: int
    mode: str
    queries: int = 0

    @property
    def avg_path_length(self):
        return float(np.mean(self.path_length))

    @property
    def pct_ir_bounces(self):
        return self.avg_path_length - 1.0


class _RenderWs:
    """Render workspaces, one per CUDA stream (launches on different streams
    may overlap)."""
    bufs = {}

    @classmethod
    def get(cls, nbytes):
        key = torch.cuda.current_stream().cuda_stream
        buf = cls.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = cls.bufs[key] = _dev.empty((max(int(nbytes), 256),), torch.uint8)
        return buf


def _c_cfg(config, scene, spp, seed, frame, cache_on, rows=None, precision=None, v1=None):
    mode = MODES[config.mode]
    c = _lib.NircRenderCfg()
    c.nbias = int(config.nbias)
    c.sph_c = float(config.sph_c)
    c.v1 = v1.data_ptr() if v1 is not None else None
    c.mode = mode
    c.spp = int(spp)
    c.cache_on = int(cache_on)
    c.max_cv = int(config.max_cache_vertices)
    if c.max_cv > 8:
        raise ConfigError("at most 8 cache vertices are supported")
    if mode >= 2:
        c.max_cv = max(c.max_cv, 1)  # one stop vertex per path (result slot 0)
    for i in range(c.max_cv):
        c.nc[i] = int(config.nc[i])
    c.rough_cut = float(config.roughness_cutoff)
    c.rr_survive = 1.0 - float(config.rr)
    c.seed = int(seed)
    c.frame = int(frame)
    c.width = int(scene.camera[14])
    c.height = int(scene.camera[15])
    r0, r1 = rows if rows is not None else (0, c.height)
    c.row0, c.row1 = int(r0), int(r1)
    c.precision = DEFAULT_PRECISION if precision is None else int(precision)
    return c


def _is_zero(cache, theta=None):
    """Cache.is_zero (caches.py:206-209) of the parameters a render will
    read: the cache's own, or the snapshot passed as ``theta`` (the frame
    pipeline trains the cache's buffer concurrently)."""
    if theta is None:
        return cache.is_zero
    lo = int(cache.spec.w_off[-1])
    return not bool(torch.any(theta[lo:] != 0).item())


def _v1_device(v1_map, w, h):
    if v1_map is None:
        return None
    a = np.ascontiguousarray(np.asarray(v1_map, np.uint8).reshape(w * h))
    return _dev.dev(a.astype(np.int32), torch.int32).to(torch.uint8)


def render_device(scene, config=None, cache=None, seed=0, spp=1, frame=0, force_cache=False,
                  rows=None, out=None, precision=None, v1_map=None, theta=None, zero=None):
    """Device-resident render: returns (img, img2, term, queries) CUDA
    tensors of sums (callers divide by spp).  ``rows`` renders a band of
    pixel rows (multi-GPU tiles); ``out`` accumulates into given buffers;
    ``v1_map`` flags the pixels where the *_sph modes may stop at the first
    vertex (estimators.py:173-217); ``theta`` renders with a snapshot buffer
    of the cache's layout instead of cache.theta."""
    if config is None:
        config = EstimatorConfig()
    mode = MODES[config.mode]
    w, h = int(scene.camera[14]), int(scene.camera[15])
    cache_on = 0
    if mode >= 1 and cache is not None and (
            force_cache or not (zero if zero is not None else _is_zero(cache, theta))):
        cache_on = 1
    v1 = _v1_device(v1_map, w, h) if mode in (3, 4) else None
    cfg = _c_cfg(config, scene, spp, seed, frame, cache_on, rows, precision, v1)
    lib = _lib.load()
    ds = scene.device()
    if out is None:
        img = _dev.zeros((h, w, 3), torch.float64)
        img2 = _dev.zeros((h, w, 3), torch.float64)
        term = _dev.zeros((h, w), torch.float64)
    else:
        img, img2, term = out
    queries = _dev.zeros((1,), torch.int64)
    ws = _RenderWs.get(lib.nirc_render_workspace_bytes(C.byref(cfg)))
    if cache_on:
        cs = _lib.make_c_spec(cache.spec)
        spec_p, theta_p = C.byref(cs), _dev.ptr(cache.theta if theta is None else theta)
    else:
        spec_p, theta_p = None, None
    _lib.check(lib.nirc_render(ds.ptr(), _dev.ptr(ds.cam), C.byref(cfg), spec_p, theta_p,
                               _dev.ptr(img), _dev.ptr(img2), _dev.ptr(term), _dev.ptr(queries),
                               _dev.ptr(ws), int(ws.numel()), _dev.stream()), "nirc_render")
    return img, img2, term, queries


def render_and_collect(scene, config, cache, seed=0, spp=1, frame=0, count=None,
                       train_frame=None, rows=None, paths=None, out=None, precision=None,
                       theta=None, defer=False, zero=None):
    """render_device + cache.collect of the same frame in ONE device pass
    (C ABI nirc_render_collect: the training walks are the first work items
    of the persistent path tracer).  Equivalent to calling render_device and
    then collect_training_records(scene, cache.seed, count, cache.record_kind,
    train_frame).  ``paths`` = (p0, p1) collects a path shard (multi-GPU).
    ``theta`` renders with another parameter buffer of the cache's layout
    (a snapshot); ``defer`` returns a callable that yields the Records once
    the launch is done instead of waiting for the record count here.
    Returns (img, img2, term, queries, Records or its callable)."""
    from .caches import Records, default_train_count
    from .records import _KIND, _check_kind, record_buffers

    if config is None:
        config = EstimatorConfig()
    mode = MODES[config.mode]
    _check_kind(scene, cache.record_kind)
    if count is None:
        count = default_train_count(scene)
    if train_frame is None:
        train_frame = frame
    p0, p1 = (0, int(count)) if paths is None else (int(paths[0]), int(paths[1]))
    w, h = int(scene.camera[14]), int(scene.camera[15])
    # ``zero``: the caller already knows Cache.is_zero of the parameters
    # (the frame pipelines read it asynchronously after training)
    if zero is None:
        zero = _is_zero(cache, theta)
    cache_on = 1 if (mode >= 1 and not zero) else 0
    cfg = _c_cfg(config, scene, spp, seed, frame, cache_on, rows, precision)
    lib = _lib.load()
    ds = scene.device()
    if out is None:
        img = _dev.zeros((h, w, 3), torch.float64)
        img2 = _dev.zeros((h, w, 3), torch.float64)
        term = _dev.zeros((h, w), torch.float64)
    else:
        img, img2, term = out
    queries = _dev.zeros((1,), torch.int64)
    n_out = _dev.zeros((1,), torch.int64)
    rec_out, ro = record_buffers(max(p1 - p0, 1))
    ws = _RenderWs.get(lib.nirc_render_collect_workspace_bytes(C.byref(cfg), max(p1 - p0, 1)))
    cs = _lib.make_c_spec(cache.spec)
    th = cache.theta if theta is None else theta
    _lib.check(lib.nirc_render_collect(
        ds.ptr(), _dev.ptr(ds.cam), C.byref(cfg), C.byref(cs) if cache_on else None,
        _dev.ptr(th) if cache_on else None, _dev.ptr(img), _dev.ptr(img2),
        _dev.ptr(term), _dev.ptr(queries), int(cache.seed), int(train_frame), p0,
        max(p1 - p0, 1), _KIND[cache.record_kind], C.byref(ro), _dev.ptr(n_out), _dev.ptr(ws),
        int(ws.numel()), _dev.stream()), "nirc_render_collect")

    def finish():
        n = int(n_out.item()) if p1 > p0 else 0
        return Records(kind=cache.record_kind, frame=train_frame, n=n,
                       **{k: v[:n] for k, v in rec_out.items()})

    return img, img2, term, queries, (finish if defer else finish())


def render(scene, config=None, cache=None, seed=0, spp=1, frame=0, v1_map=None,
           force_cache=False, precision=None):
    """Render with the configured estimator (estimators.py:173-217)."""
    if config is None:
        config = EstimatorConfig()
    if v1_map is not None and MODES[config.mode] <= 1:
        v1_map = None  # only the *_sph modes read it
    img, img2, term, queries = render_device(scene, config, cache, seed, spp, frame,
                                             force_cache, precision=precision, v1_map=v1_map)
    img = img.cpu().numpy()
    img2 = img2.cpu().numpy()
    term = term.cpu().numpy()
    mean = img / spp
    if spp > 1:
        var = (img2 - img * img / spp) / (spp - 1)
        np.maximum(var, 0.0, out=var)
    else:
        var = np.zeros_like(img)
    return RenderResult(mean, var, term / spp, spp, config.mode, int(queries.item()))


def render_two_level(scene, cache, seed=0, spp=1, frame=0, config=None, force_cache=False):
    """Cache-plus-residual render; any cache state keeps the mean."""
    if config is None:
        config = EstimatorConfig(mode="two-level")
    if config.mode != "two-level":
        raise ConfigError(f"config mode '{config.mode}' is not two-level")
    return render(scene, config, cache, seed, spp, frame, force_cache=force_cache)


def render_biased(scene, cache, config, seed=0, spp=1, frame=0, v1_map=None):
    """Early-stop render shading stop vertices from the cache
    (estimators.py:231-237)."""
    if not config.mode.startswith("biased-"):
        raise ConfigError(f"config mode '{config.mode}' is not biased")
    return render(scene, config, cache, seed, spp, frame, v1_map=v1_map, force_cache=True)


# ---- per-interaction estimators and helpers (estimators.py:86-136, 240-320,
# 386-393 of the reference) -------------------------------------------------
@dataclass
class PathState:
    """Per-path bookkeeping of the biased stop tests (estimators.py:86-95)."""

    throughput: np.ndarray = None
    vertex: int = 0
    a: float = 1.0
    a0: float = 0.0
    alive: bool = True
    prev_pdf: float = -1.0

    def __post_init__(self):
        if self.throughput is None:
            self.throughput = np.ones(3)


def sph_update(state, seg_len, pdf, cos_arrival):
    """Fold one traced segment into the footprint state (estimators.py:98-118):
    the first segment sets a0, later ones scale a by (len / (pdf cos))^2."""
    import math
    from dataclasses import replace

    s = replace(state, vertex=state.vertex + 1, prev_pdf=pdf)
    if cos_arrival <= 0.0:
        s.a = math.inf
        return s
    if state.vertex == 0:
        s.a0 = seg_len * seg_len / (4.0 * math.pi * cos_arrival)
        return s
    if pdf > 0.0:
        f = seg_len / (pdf * cos_arrival)
        s.a = state.a * f * f
    return s


def sph_should_terminate(state, c=0.01):
    """Spread test: fires from the second bounce once a > c * a0."""
    return state.vertex >= 2 and state.a > c * state.a0


def bth_continuation_probability(pdf, n_cache):
    """Survival probability pdf / (pdf + n_cache / pi) of the stochastic
    brdf test (estimators.py:126-136)."""
    import math

    if pdf < 0.0 or not math.isfinite(pdf):
        raise ConfigError(f"pdf {pdf} must be finite and non-negative")
    if n_cache < 1:
        raise ConfigError("n_cache must be at least 1")
    return pdf / (pdf + n_cache / math.pi)


def _surface_dirs(scene, it, n, seed, stream, offset):
    """n brdf draws at an interaction, (dirs, pdf, f, cos) with invalid rows
    zero (estimators.py:260-278): u from the P_MEASURE stream (host rng,
    bit-exact), the BSDF sampling on the device."""
    from .rng import P_MEASURE, uniform_array

    u = _dev.dev(uniform_array(seed, P_MEASURE, stream, 2 * n, offset=offset), torch.float64)
    dirs = _dev.zeros((n, 3), torch.float64)
    pdf = _dev.zeros((n,), torch.float64)
    fval = _dev.zeros((n, 3), torch.float64)
    cos = _dev.zeros((n,), torch.float64)
    ns = np.ascontiguousarray(np.asarray(it.ns, np.float64))
    wo = np.ascontiguousarray(np.asarray(it.wo, np.float64))
    lib = _lib.load()
    ds = scene.device()
    _lib.check(lib.nirc_surface_samples(ds.ptr(), ns.ctypes.data, wo.ctypes.data, int(it.mat),
                                        _dev.ptr(u), int(n), _dev.ptr(dirs), _dev.ptr(pdf),
                                        _dev.ptr(fval), _dev.ptr(cos), _dev.stream()),
               "nirc_surface_samples")
    return dirs.cpu().numpy(), pdf.cpu().numpy(), fval.cpu().numpy(), cos.cpu().numpy()


def _check_not_delta(scene, it, what):
    from .scene import MAT_MIRROR

    if int(scene.pack.mat_kind[it.mat]) == MAT_MIRROR:
        raise ConfigError(f"{what} undefined on a delta lobe")


def estimate_Lc(scene, it, cache, n_c=15, seed=0, stream=0):
    """Cache term of the two-level split at one interaction
    (estimators.py:281-296): mean over n_c brdf-sampled directions of
    n(w) f cos / pdf; rejected draws contribute zero."""
    _check_not_delta(scene, it, "cache term")
    if n_c < 1:
        raise ConfigError("n_c must be at least 1")
    dirs, pdf, fval, cos = _surface_dirs(scene, it, n_c, seed, stream, 0)
    out = np.zeros(3)
    ok = pdf > 0.0
    if np.any(ok):
        pred = cache.nirc_query(it, dirs[ok])
        wgt = cos[ok] / pdf[ok]
        out = np.sum(pred * fval[ok] * wgt[:, None], axis=0)
    return out / n_c


def estimate_Lr(scene, it, cache, n_r=1, seed=0, stream=0):
    """Residual term of the split (estimators.py:299-320): mean over n_r
    fresh brdf draws of (L_i(w) - n(w)) f cos / pdf, L_i from an
    independent device recording walk along w."""
    from .caches import sample_incident_targets

    _check_not_delta(scene, it, "residual term")
    if n_r < 1:
        raise ConfigError("n_r must be at least 1")
    dirs, pdf, fval, cos = _surface_dirs(scene, it, n_r, seed, stream, 1000)
    out = np.zeros(3)
    for k in range(n_r):
        if pdf[k] <= 0.0:
            continue
        li, _ = sample_incident_targets(scene, it.position, dirs[k], seed + 7919 * (stream + 1),
                                        1, prev_pdf=pdf[k], prev_ns=it.ns, frame=k)
        pred = cache.nirc_query(it, dirs[k][None, :])[0]
        out += (li[0] - pred) * fval[k] * (cos[k] / pdf[k])
    return out / n_r


def estimate_env_direct(scene, cache, it, n_c=15, n_r=1, seed=0, stream=0):
    """Two-level estimate of reflected direct environment light at one
    interaction (estimators.py:323-348): the cache's per-direction
    prediction (a visibility cache scaled by the known environment radiance)
    over n_c brdf draws, plus n_r shadow-rayed residual draws (device
    occlusion queries, nirc_occluded)."""
    if scene.pack.env_kind == 0:
        raise ConfigError("scene has no environment light")
    dirs, pdf, fval, cos = _surface_dirs(scene, it, n_c, seed, stream, 0)
    out = np.zeros(3)
    ok = pdf > 0.0
    if np.any(ok):
        pred = _env_prediction(scene, cache, it, dirs[ok])
        wgt = cos[ok] / pdf[ok]
        out += np.sum(pred * fval[ok] * wgt[:, None], axis=0) / n_c
    dirs, pdf, fval, cos = _surface_dirs(scene, it, n_r, seed, stream, 1000)
    ok = pdf > 0.0
    if np.any(ok):
        pred = _env_prediction(scene, cache, it, dirs[ok])
        shadow = _shadowed(scene, it, dirs[ok])
        true = np.zeros_like(pred)
        for j, d in enumerate(dirs[ok]):
            if not shadow[j]:
                true[j] = scene.env_radiance(d)
        wgt = cos[ok] / pdf[ok]
        out += np.sum((true - pred) * fval[ok] * wgt[:, None], axis=0) / n_r
    return out


def _env_prediction(scene, cache, it, dirs):
    """estimators.py:351-356."""
    if cache.kind == "nvc":
        vis = cache.nvc_query(it, dirs)
        env = np.array([scene.env_radiance(d) for d in dirs])
        return vis * env
    return cache.nirc_query(it, dirs)


def _shadowed(scene, it, wis):
    """estimators.py:359-370 for a batch of directions: shadow rays spawned
    eps along the side of the geometric normal facing each direction, any-hit
    to T_FAR on the device."""
    wis = np.atleast_2d(np.asarray(wis, np.float64))
    n = wis.shape[0]
    p, g = np.asarray(it.position, float), np.asarray(it.ng, float)
    eps = float(scene.pack.eps)
    org = np.empty((n, 3))
    for k in range(n):
        sgn = 1.0 if float(g @ wis[k]) > 0.0 else -1.0
        org[k] = (p[0] + sgn * eps * g[0], p[1] + sgn * eps * g[1], p[2] + sgn * eps * g[2])
    o_d, d_d = _dev.dev(org, torch.float64), _dev.dev(np.ascontiguousarray(wis), torch.float64)
    res = _dev.zeros((n,), torch.uint8)
    ds = scene.device()
    lib = _lib.load()
    _lib.check(lib.nirc_occluded(ds.ptr(), _dev.ptr(o_d), _dev.ptr(d_d), n, T_FAR, _dev.ptr(res),
                                 _dev.stream()), "nirc_occluded")
    return res.cpu().numpy().astype(bool)


def pt_radiance(scene, ix, iy, seed=0, sample=0, frame=0):
    """One path-traced radiance sample of pixel (ix, iy) as the renderer
    draws it (estimators.py:240-257), traced on the device."""
    cfg = _c_cfg(EstimatorConfig(mode="pt"), scene, 1, seed, frame, 0)
    out = _dev.zeros((3,), torch.float64)
    lib = _lib.load()
    ds = scene.device()
    _lib.check(lib.nirc_pt_radiance(ds.ptr(), _dev.ptr(ds.cam), C.byref(cfg), int(ix), int(iy),
                                    int(sample), _dev.ptr(out), _dev.stream()),
               "nirc_pt_radiance")
    return out.cpu().numpy()


def reference_render(scene, spp, seed=0, out_dir=".refcache", allow_compute=True, force=False):
    """Path-traced reference image, cached on disk as PFM by scene state and
    seed (estimators.py:386-393)."""
    import os

    from .pfm import read_pfm, write_pfm

    path = os.path.join(out_dir, f"ref-{scene.content_hash()}-{spp}-{seed}.pfm")
    if not force and os.path.exists(path):
        return read_pfm(path).astype(np.float64)
    if not allow_compute:
        raise ConfigError(f"missing cached render {path}")
    img = render(scene, EstimatorConfig(mode="pt"), seed=seed, spp=spp).image
    os.makedirs(out_dir, exist_ok=True)
    write_pfm(path, img)
    return np.asarray(img, np.float64)
