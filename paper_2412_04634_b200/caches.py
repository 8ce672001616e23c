"""Neural caches and their online training on the B200 (drop-in for
pkg/src/nirclab/caches.py).

θ, the Adam moments and the training records live in device memory.
``train_frame`` is one C-ABI ``nirc_train_frame`` call: the batches of all
steps from the splitmix64 shuffle stream, then per optimizer step the fused
encode / forward / loss / backward + hash-grid scatter kernel and dense Adam;
it synchronises with the host once per frame to read the loss trace and the
status flags.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import tempfile
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .adam import AdamState
from .errors import ConfigError, DivergenceError, InvalidSampleError
from .mlp import ACT_RELU, ACT_SIGMOID, init_theta, make_spec

KINDS = ("nirc", "nrc", "nvc")
RECORD_KINDS = ("nirc", "nrc", "nvc", "nirc_full", "nirc_env")
LOSS_KINDS = ("l2", "relative_l2", "variance", "bce")
BATCH_CAP = 16384
EMA_ALPHA = 0.95


@dataclass
class Records:
    """One frame of training data (caches.py:38-53).  Arrays may be numpy
    or CUDA tensors; ``device()`` returns the f64 CUDA view the kernels use."""

    kind: str
    pos: object
    ns: object
    alb: object
    rough: object
    dirs: object
    target: object
    pdf: object
    frame: int
    n: int = None
    _dev_cache: dict = field(default=None, repr=False)

    def __len__(self):
        if self.n is not None:
            return int(self.n)
        return int(self.pos.shape[0])

    def device(self):
        if self._dev_cache is None:
            n = len(self)
            self._dev_cache = {k: _dev.dev(getattr(self, k), torch.float64)[:n].contiguous()
                               for k in ("pos", "ns", "alb", "rough", "dirs", "target", "pdf")}
        return self._dev_cache

    def c_struct(self):
        d = self.device()
        r = _lib.NircRecords()
        for k, t in d.items():
            setattr(r, k, t.data_ptr())
        r.n = len(self)
        return r, d


def default_train_count(scene, fraction=0.025):
    """ceil(fraction * W * H) training paths (caches.py:80-84)."""
    w = int(scene.camera[14])
    h = int(scene.camera[15])
    return max(1, int(math.ceil(fraction * w * h)))


class _Workspace:
    """Cached device workspace, grown on demand."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes):
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = _dev.empty((max(int(nbytes), 256),), torch.uint8)
        return self.buf


@dataclass
class TrainResult:
    trace: list
    adam: AdamState
    batch_idx: list = None
    flags: int = 0
    diverged_step: int = -1


def _launch_steps(spec, theta, adam, records, seed, frame, steps, batch, loss_kind, loss_eps,
                  running_mean, ws, return_idx=False, deterministic=False):
    n = len(records)
    if n == 0:
        raise ValueError("cannot train on an empty record set")
    cap = BATCH_CAP if batch is None else int(batch)
    if cap < 1:
        raise ValueError(f"batch must be positive, got {batch}")
    lib = _lib.load()
    cs = _lib.make_c_spec(spec)
    rec, _keep = records.c_struct()
    B = min(cap, n)
    losses = _dev.zeros((steps,), torch.float64)
    flags = _dev.zeros((1,), torch.int32)
    opts = C.byref(_lib.train_opts(adam, deterministic))
    idx = None
    if not return_idx:
        # one C call: batches of all steps selected at once, then the steps
        need = lib.nirc_train_frame_workspace_bytes(cs, n, cap, steps)
        buf = ws.get(need)
        _lib.check(lib.nirc_train_frame(
            cs, _dev.ptr(theta), _dev.ptr(adam.m), _dev.ptr(adam.v), _dev.ptr(adam._t),
            _dev.ptr(adam._skipped), rec, int(seed), int(frame), int(steps), cap,
            LOSS_KINDS.index(loss_kind), float(loss_eps), float(adam.lr), opts,
            _dev.ptr(running_mean), _dev.ptr(losses), _dev.ptr(flags), _dev.ptr(buf),
            int(buf.numel()), _dev.stream()), "nirc_train_frame")
    else:
        need = lib.nirc_train_workspace_bytes(cs, n, cap)
        buf = ws.get(need)
        idx = [_dev.empty((B,), torch.int64) for _ in range(steps)]
        for s in range(steps):
            _lib.check(lib.nirc_train_step(
                cs, _dev.ptr(theta), _dev.ptr(adam.m), _dev.ptr(adam.v), _dev.ptr(adam._t),
                _dev.ptr(adam._skipped), rec, int(seed), int(frame), s, cap,
                LOSS_KINDS.index(loss_kind), float(loss_eps), float(adam.lr), opts,
                _dev.ptr(running_mean), _dev.ptr(losses[s:s + 1]), _dev.ptr(flags),
                _dev.ptr(idx[s]), _dev.ptr(buf), int(buf.numel()), _dev.stream()),
                "nirc_train_step")
    trace = losses.cpu().numpy().tolist()
    f = int(flags.item())
    res = TrainResult(trace=trace, adam=adam, flags=f)
    if return_idx:
        res.batch_idx = [i.cpu().numpy() for i in idx]
    if f & 2:
        res.diverged_step = next(i for i, v in enumerate(trace) if not math.isfinite(v))
    return res


def collect_training_records(scene, seed, count, kind="nirc", frame=0):
    """Trace `count` camera paths and distill records of the given kind
    (caches.py:87-131), on the device (records.py)."""
    from .records import collect_training_records as _collect

    return _collect(scene, seed, count, kind, frame)


def sample_incident_targets(scene, origin, direction, seed, count, prev_pdf=-1.0,
                            prev_ns=(0.0, 0.0, 0.0), frame=0):
    """Independent incident-radiance estimates along one fixed ray
    (caches.py:134-155): (targets, full_targets), each (count, 3), from
    `count` device walk_record walks (C ABI nirc_incident_targets)."""
    count = int(count)
    out = _dev.zeros((max(count, 1), 3), torch.float64)
    out_full = _dev.zeros((max(count, 1), 3), torch.float64)
    if count > 0:
        o = np.ascontiguousarray(np.asarray(origin, np.float64).reshape(3))
        d = np.ascontiguousarray(np.asarray(direction, np.float64).reshape(3))
        pn = np.ascontiguousarray(np.asarray(prev_ns, np.float64).reshape(3))
        ds = scene.device()
        lib = _lib.load()
        _lib.check(lib.nirc_incident_targets(
            ds.ptr(), int(seed), int(frame), o.ctypes.data, d.ctypes.data, float(prev_pdf),
            pn.ctypes.data, count, _dev.ptr(out), _dev.ptr(out_full), _dev.stream()),
            "nirc_incident_targets")
    return out[:count].cpu().numpy(), out_full[:count].cpu().numpy()


def train_frame_device(spec, theta, records, seed, frame, steps=4, batch=None, adam=None,
                       loss_kind="relative_l2", loss_eps=0.01, return_idx=False,
                       deterministic=False):
    """Device training on a bare (spec, theta) pair -- the batch form of
    train_frame used by tests and the benchmark.  ``deterministic`` sums the
    hash-grid gradient in np.add.at's order (bit-reproducible runs)."""
    if adam is None:
        adam = AdamState(theta)
    rm = _dev.zeros((3,), torch.float64)
    return _launch_steps(spec, theta, adam, records, seed, frame, steps, batch, loss_kind,
                         loss_eps, rm, _Workspace(), return_idx, deterministic)


class Cache:
    """A neural cache bound to one scene: device θ plus optimizer state
    (caches.py:158-298)."""

    def __init__(self, kind, scene, spec, theta, adam, loss_kind, record_kind, seed):
        self.kind = kind
        self.scene = scene
        self.spec = spec
        self.theta = _dev.dev(theta, torch.float32).clone()
        self.adam = adam
        self.loss_kind = loss_kind
        self.record_kind = record_kind
        self.seed = int(seed)
        self.frame = 0
        self.loss_eps = 0.01
        self._running_mean = _dev.zeros((3,), torch.float64)
        self.snapshot_dir = None
        self.has_env = scene.pack.env_kind != 0
        self._ws = _Workspace()
        # bit-reproducible training (ordered grid-gradient scatter) -- the
        # reference's contract; NIRC_DETERMINISTIC=0 trades it
        # for the atomic scatter
        self.deterministic = os.environ.get("NIRC_DETERMINISTIC", "1") != "0"

    @property
    def running_mean(self):
        return self._running_mean.cpu().numpy()

    @running_mean.setter
    def running_mean(self, value):
        self._running_mean.copy_(torch.as_tensor(np.asarray(value, np.float64)))

    @classmethod
    def create(cls, kind, scene, seed=0, loss=None, record_kind=None, init="zero", levels=12,
               table_log2=15, feats=2, bands=4, depth=4, width=64, lr=0.01):
        if kind not in KINDS:
            raise ConfigError(f"unknown cache kind '{kind}'")
        if loss is None:
            loss = "bce" if kind == "nvc" else "relative_l2"
        if loss not in LOSS_KINDS:
            raise ConfigError(f"unknown loss '{loss}'")
        if record_kind is None:
            record_kind = kind
        if record_kind not in RECORD_KINDS:
            raise ConfigError(f"unknown record kind '{record_kind}'")
        pack = scene.pack
        bb_min = np.array(pack.bbox_min, float)
        bb_ext = 1.0 / np.array(pack.bbox_inv_ext, float)
        spec = make_spec(levels=levels, table=1 << table_log2, feats=feats, bands=bands,
                         depth=depth, width=width, out_dim=3,
                         out_act=ACT_SIGMOID if kind == "nvc" else ACT_RELU,
                         bb_min=bb_min, bb_ext=bb_ext)
        theta = init_theta(spec, seed=seed, out_scale=0.05 if init == "random" else 0.0)
        adam = AdamState(theta, lr=lr)
        return cls(kind, scene, spec, theta, adam, loss, record_kind, seed)

    @property
    def is_zero(self):
        """Last layer W and b all zero => the net predicts exactly 0
        (caches.py:206-209)."""
        lo = int(self.spec.w_off[-1])
        return not bool(torch.any(self.theta[lo:] != 0).item())

    def theta_host(self):
        return self.theta.cpu().numpy()

    # -- queries ---------------------------------------------------------
    def _query(self, surface, dirs):
        """caches.py:211-233: one surface, N directions (C ABI nirc_query)."""
        from .mlp import query

        pack = self.scene.pack
        m = surface.mat
        dirs = np.atleast_2d(np.asarray(dirs, float))
        surf = np.concatenate([np.asarray(surface.position, float), np.asarray(surface.ns, float),
                               np.asarray(pack.mat_albedo[m], float),
                               [float(pack.mat_rough[m])]])[None, :]
        y = query(self.spec, self.theta, surf, dirs, np.zeros(dirs.shape[0], np.int32))
        return np.asarray(y, np.float64)

    def nirc_query(self, surface, dirs):
        """Predicted incident indirect radiance per direction, (N, 3)."""
        return self._query(surface, dirs)

    def nrc_query(self, surface, wo=None):
        if wo is None:
            wo = surface.wo
        return self._query(surface, np.asarray(wo, float)[None, :])[0]

    def nvc_query(self, surface, dirs):
        if not self.has_env:
            raise ConfigError("visibility cache queried on a scene without an environment light")
        return self._query(surface, dirs)

    # -- training --------------------------------------------------------
    def collect(self, count=None, frame=None):
        from .records import collect_training_records

        if count is None:
            count = default_train_count(self.scene)
        if frame is None:
            frame = self.frame
        return collect_training_records(self.scene, self.seed, count, self.record_kind, frame)

    def train_frame(self, records, steps=4):
        return train_frame(self, records, steps)

    # -- snapshots -------------------------------------------------------
    def save(self, path):
        from .snapshot import save_snapshot

        st = self.adam
        save_snapshot(path, {
            "theta": self.theta_host(), "m": st.m.cpu().numpy(), "v": st.v.cpu().numpy(),
            "t": np.int64(st.t), "frame": np.int64(self.frame),
            "running_mean": self.running_mean,
            "kind": np.int64(KINDS.index(self.kind)),
            "loss": np.int64(LOSS_KINDS.index(self.loss_kind)),
            "record": np.int64(RECORD_KINDS.index(self.record_kind)),
            "seed": np.int64(self.seed), "lr": np.float64(st.lr),
            "net": np.array([self.spec.levels, self.spec.table, self.spec.feats,
                             self.spec.bands, len(self.spec.dims) - 2, self.spec.dims[1]],
                            np.int64),
            "bb_min": np.asarray(self.spec.bb_min, float),
            "bb_ext": 1.0 / np.asarray(self.spec.bb_inv, float),
        })

    @classmethod
    def load(cls, path, scene):
        from .snapshot import load_snapshot

        d = load_snapshot(path)
        net = d["net"]
        kind = KINDS[int(d["kind"])]
        spec = make_spec(levels=int(net[0]), table=int(net[1]), feats=int(net[2]),
                         bands=int(net[3]), depth=int(net[4]), width=int(net[5]), out_dim=3,
                         out_act=ACT_SIGMOID if kind == "nvc" else ACT_RELU,
                         bb_min=d["bb_min"], bb_ext=d["bb_ext"])
        theta = d["theta"].copy()
        adam = AdamState(theta, lr=float(d["lr"]))
        adam.m.copy_(torch.from_numpy(d["m"].astype(np.float32)))
        adam.v.copy_(torch.from_numpy(d["v"].astype(np.float32)))
        adam.t = int(d["t"])
        cache = cls(kind, scene, spec, theta, adam, LOSS_KINDS[int(d["loss"])],
                    RECORD_KINDS[int(d["record"])], int(d["seed"]))
        cache.frame = int(d["frame"])
        cache.running_mean = d["running_mean"]
        return cache


def _dump_diagnostics(cache, step, value):
    out_dir = cache.snapshot_dir or tempfile.gettempdir()
    path = os.path.join(out_dir, f"diverged_{cache.kind}_frame{cache.frame}.nncache")
    cache.save(path)
    return (f"non-finite loss ({value}) at frame {cache.frame} step {step}; "
            f"state dumped to {path}"), path


def train_frame(cache, records, steps=4, batch=None):
    """`steps` optimizer updates on one frame of records (caches.py:310-354).
    Returns the per-step loss trace; raises DivergenceError (after dumping
    the state) on a non-finite loss, InvalidSampleError on pdf <= 0."""
    if len(records) == 0:
        raise ValueError("cannot train on an empty record set")
    res = _launch_steps(cache.spec, cache.theta, cache.adam, records, cache.seed, cache.frame,
                        steps, batch, cache.loss_kind, cache.loss_eps, cache._running_mean,
                        cache._ws, deterministic=getattr(cache, "deterministic", False))
    if res.flags & 1:
        raise InvalidSampleError("sample pdf must be positive")
    if res.flags & 2:
        s = res.diverged_step
        msg, path = _dump_diagnostics(cache, s, res.trace[s])
        raise DivergenceError(msg, snapshot_path=path)
    cache.frame += 1
    return res.trace
