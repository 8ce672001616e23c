"""Multi-GPU NIRC frame: pixel-row bands, path shards and one gradient
all-reduce per optimizer step.

The reference is single-threaded (pkg/src/nirclab/experiment.py:1-8); every
random draw it makes is addressed by (seed, purpose, frame, pixel|path,
sample, dim) (pkg/src/nirclab/rng.py:59-106), so a frame partitions exactly:

* render  -- rank r traces the pixel rows ``split_range(H, world, r)``
  (render_kernel, kernels.py:723-759, keys stream_key(seed, P_RENDER, frame,
  pix, s)); the union of the bands is bit-identical to a 1-GPU render and
  needs no communication.
* collect -- rank r walks the training paths ``split_range(count, world,
  r)`` (collect_paths_kernel, kernels.py:289-311, keys stream_key(seed,
  P_TRAIN, frame, p, 0)); the records are all-gathered in rank order, which
  reproduces the reference's path-major row order exactly.
* train   -- every rank selects the same batch (caches.py:327-329) and runs
  the fused encode/forward/loss/backward over its share of the 128-row batch
  tiles; the flat gradient (theta_len f32) and [loss sum, bad-pdf] are
  summed with one all-reduce each; every rank then runs the identical dense
  Adam, so the cache replicas stay bit-identical (all-reduce results are
  identical on every rank).

One process per GPU, torch.distributed for the plumbing (NCCL over NVLink on
the B200 box, gloo in the CPU tests).  The per-rank compute goes through an
``ops`` object: ``DeviceOps`` calls the C ABI (include/nirc_b200.h); the CPU
tests substitute a checker built on the oracle to exercise this host logic.
"""

from __future__ import annotations

import ctypes as C
import math

import torch

from .errors import DivergenceError, InvalidSampleError

REC_COLS = (("pos", 3), ("ns", 3), ("alb", 3), ("rough", 1), ("dirs", 3), ("target", 3),
            ("pdf", 1))
REC_WIDTH = sum(w for _, w in REC_COLS)  # 17 f64 per record
FUSED_LOSSES = ("l2", "relative_l2")


def split_range(n, world, rank):
    """Contiguous balanced shard [lo, hi) of range(n) for `rank`."""
    n, world, rank = int(n), int(world), int(rank)
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_records(cols):
    """(n, 17) f64 tensor from a dict of record columns (REC_COLS order)."""
    n = int(cols["pos"].shape[0])
    return torch.cat([cols[k].reshape(n, w) for k, w in REC_COLS], dim=1)


def unpack_records(packed, kind, frame):
    from .caches import Records

    out, c = {}, 0
    for k, w in REC_COLS:
        v = packed[:, c:c + w]
        out[k] = (v.reshape(-1) if w == 1 else v).contiguous()
        c += w
    return Records(kind=kind, frame=frame, n=int(packed.shape[0]), **out)


class Comm:
    """torch.distributed over one process group (rank order = shard order)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo (CPU tests, shared-GPU tests) all-gathers host tensors only
        self.host_gather = dist.get_backend(group) == "gloo"

    def all_reduce_sum_(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_reduce_max_(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def barrier(self):
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def broadcast_(self, t, src=0):
        if self.world > 1:
            self.dist.broadcast(t, src=src, group=self.group)
        return t

    def all_gather_rows(self, t):
        """Concatenate every rank's rows (any count, same trailing shape) in
        rank order.  One host read of the row counts."""
        if self.world == 1:
            return t
        if self.host_gather and t.is_cuda:
            return self._gather_rows(t.cpu()).to(t.device)
        return self._gather_rows(t)

    def _gather_rows(self, t):
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        counts = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(counts, n, group=self.group)
        counts = torch.cat(counts).tolist()  # one host read for all ranks' counts
        mx = max(counts)
        if mx == 0:
            return t[:0]
        pad = t.new_zeros((mx,) + tuple(t.shape[1:]))
        pad[: t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(bufs, pad, group=self.group)
        return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


class DeviceOps:
    """The per-rank compute of the sharded frame through the C ABI."""

    def __init__(self):
        from . import _lib

        self.lib = _lib.load()
        self._ws = {}

    def _buf(self, key, nbytes):
        from . import _dev

        b = self._ws.get(key)
        if b is None or b.numel() < nbytes:
            b = _dev.empty((max(int(nbytes), 256),), torch.uint8)
            self._ws[key] = b
        return b

    def collect_range(self, scene, seed, frame, path0, count, kind):
        """Records of training paths [path0, path0+count) as a packed
        (n, 17) f64 CUDA tensor (nirc_collect_range)."""
        from . import _dev, _lib
        from .records import _KIND

        if count <= 0:
            return _dev.empty((0, REC_WIDTH), torch.float64)
        cap = int(count) * 63
        cols = {k: _dev.empty((cap, w) if w > 1 else (cap,), torch.float64) for k, w in REC_COLS}
        ro = _lib.NircRecordsOut()
        for k, t in cols.items():
            setattr(ro, k, t.data_ptr())
        ro.cap = cap
        n_out = _dev.zeros((1,), torch.int64)
        ws = self._buf("collect", self.lib.nirc_collect_workspace_bytes(int(count)))
        ds = scene.device()
        _lib.check(self.lib.nirc_collect_range(
            ds.ptr(), _dev.ptr(ds.cam), int(seed), int(frame), int(path0), int(count),
            _KIND[kind], C.byref(ro), _dev.ptr(n_out), _dev.ptr(ws), int(ws.numel()),
            _dev.stream()), "nirc_collect_range")
        n = int(n_out.item())
        return pack_records({k: v[:n] for k, v in cols.items()})

    def train_tiles(self, n_records, batch_cap):
        return int(self.lib.nirc_train_tiles(int(n_records), int(batch_cap)))

    def train_grad(self, cache, records, step, batch_cap, tile_begin, tile_end, grad, aux,
                   flags):
        from . import _dev, _lib
        from .caches import LOSS_KINDS

        cs = _lib.make_c_spec(cache.spec)
        rec, _keep = records.c_struct()
        ws = self._buf("train", self.lib.nirc_train_workspace_bytes(cs, len(records),
                                                                    int(batch_cap)))
        _lib.check(self.lib.nirc_train_grad(
            cs, _dev.ptr(cache.theta), rec, int(cache.seed), int(cache.frame), int(step),
            int(batch_cap), LOSS_KINDS.index(cache.loss_kind), float(cache.loss_eps),
            C.byref(_lib.train_opts(cache.adam, getattr(cache, "deterministic", False))),
            int(tile_begin), int(tile_end), _dev.ptr(grad), _dev.ptr(aux), _dev.ptr(flags),
            None, _dev.ptr(ws), int(ws.numel()), _dev.stream()), "nirc_train_grad")

    def train_apply(self, cache, grad, aux, batch, loss_out, flags):
        from . import _dev, _lib

        st = cache.adam
        cs = _lib.make_c_spec(cache.spec)
        _lib.check(self.lib.nirc_train_apply(
            cs, _dev.ptr(cache.theta), _dev.ptr(st.m), _dev.ptr(st.v), _dev.ptr(st._t),
            _dev.ptr(st._skipped), _dev.ptr(grad), _dev.ptr(aux), int(batch), float(st.lr),
            C.byref(_lib.train_opts(st)), _dev.ptr(loss_out), _dev.ptr(flags),
            _dev.ptr(st._scratch), _dev.stream()),
            "nirc_train_apply")

    def train_full(self, cache, records, steps, batch):
        """Un-sharded steps (losses outside the fused path)."""
        from .caches import _launch_steps

        return _launch_steps(cache.spec, cache.theta, cache.adam, records, cache.seed,
                             cache.frame, steps, batch, cache.loss_kind, cache.loss_eps,
                             cache._running_mean, cache._ws)


def collect_sharded(cache, comm, count=None, frame=None, ops=None):
    """collect_training_records split by path index over the ranks; every
    rank returns the full record set in the reference's row order."""
    from .caches import default_train_count

    ops = ops or DeviceOps()
    if count is None:
        count = default_train_count(cache.scene)
    if frame is None:
        frame = cache.frame
    p0, p1 = split_range(count, comm.world, comm.rank)
    local = ops.collect_range(cache.scene, cache.seed, frame, p0, p1 - p0, cache.record_kind)
    return unpack_records(comm.all_gather_rows(local), cache.record_kind, frame)


def train_frame_sharded(cache, records, comm, steps=4, batch=None, ops=None):
    """train_frame (caches.py:310-354) with the batch tiles split over the
    ranks and the gradient all-reduced before the identical Adam step.
    Returns the loss trace; raises like train_frame."""
    from .caches import BATCH_CAP, _dump_diagnostics

    ops = ops or DeviceOps()
    n = len(records)
    if n == 0:
        raise ValueError("cannot train on an empty record set")
    cap = BATCH_CAP if batch is None else int(batch)
    if cap < 1:
        raise ValueError(f"batch must be positive, got {batch}")
    B = min(cap, n)
    theta = cache.theta
    if cache.loss_kind not in FUSED_LOSSES:
        # replicated steps, then rank 0's state is authoritative
        res = ops.train_full(cache, records, steps, batch)
        for t in (cache.theta, cache.adam.m, cache.adam.v, cache.adam._t, cache.adam._skipped,
                  cache._running_mean):
            comm.broadcast_(t, 0)
        trace, flags = res.trace, res.flags
    else:
        ntiles = ops.train_tiles(n, cap)
        t0, t1 = split_range(ntiles, comm.world, comm.rank)
        # ONE all-reduce per step: the flat gradient with [loss sum, bad-pdf
        # count] appended as two more f32 (the loss sum rounds to f32 before
        # the cross-GPU sum; every rank receives the same bits)
        plen = int(theta.numel())
        buf = torch.empty((plen + 2,), dtype=torch.float32, device=theta.device)
        grad = buf[:plen]
        aux = torch.zeros((2,), dtype=torch.float64, device=theta.device)
        flags_t = torch.zeros((1,), dtype=torch.int32, device=theta.device)
        losses = torch.zeros((steps,), dtype=torch.float64, device=theta.device)
        for s in range(steps):
            ops.train_grad(cache, records, s, cap, t0, t1, grad, aux, flags_t)
            buf[plen:].copy_(aux)
            comm.all_reduce_sum_(buf)
            aux.copy_(buf[plen:])
            ops.train_apply(cache, grad, aux, B, losses[s:s + 1], flags_t)
        trace = losses.cpu().numpy().tolist()
        flags = int(flags_t.item())
    if flags & 1:
        raise InvalidSampleError("sample pdf must be positive")
    if flags & 2:
        s = next(i for i, v in enumerate(trace) if not math.isfinite(v))
        path = None
        if comm.rank == 0:
            msg, path = _dump_diagnostics(cache, s, trace[s])
        else:
            msg = f"non-finite loss ({trace[s]}) at frame {cache.frame} step {s} (rank {comm.rank})"
        raise DivergenceError(msg, snapshot_path=path)
    cache.frame += 1
    return trace


def render_band(scene, config, cache, comm, seed=0, spp=1, frame=0, out=None):
    """This rank's pixel-row band of render/render_two_level: device sums
    (img, img2, term) of the full frame shape with only rows [r0, r1)
    written, the executed-query counter and the band."""
    from .estimators import render_device

    h = int(scene.camera[15])
    rows = split_range(h, comm.world, comm.rank)
    if rows[1] <= rows[0]:
        raise ValueError(f"rank {comm.rank} has no pixel rows ({h} rows over {comm.world})")
    img, img2, term, q = render_device(scene, config, cache, seed, spp, frame, rows=rows, out=out)
    return img, img2, term, q, rows


def gather_image(t, rows, comm):
    """All-gather the row bands of a (H, W, ...) device image into the full
    frame on every rank (the optional reporting exchange)."""
    band = t[rows[0]:rows[1]].contiguous()
    full = comm.all_gather_rows(band)
    return full


def run_frame_sharded(scene, cache, config, comm, seed, frame, spp=1, steps=4, batch=None,
                      train_fraction=0.025, out=None, ops=None):
    """One frame of the online two-level renderer on `comm.world` GPUs:
    render this rank's row band with θ_f and walk its training-path shard in
    the same trace launch (nirc_render_collect), all-gather the records and
    train with all-reduced gradients (θ_{f+1} on every rank).
    Returns ((img, img2, term) band sums, rows, stats dict)."""
    from .caches import default_train_count
    from .estimators import render_and_collect

    if cache is None:
        img, img2, term, q, rows = render_band(scene, config, cache, comm, seed, spp, frame, out)
        return (img, img2, term), rows, {"rows": rows, "queries": q}
    h = int(scene.camera[15])
    rows = split_range(h, comm.world, comm.rank)
    count = default_train_count(scene, train_fraction)
    paths = split_range(count, comm.world, comm.rank)
    img, img2, term, q, local = render_and_collect(scene, config, cache, seed, spp, frame,
                                                   count=count, rows=rows, paths=paths, out=out)
    packed = pack_records({k: getattr(local, k) for k, _ in REC_COLS})
    rec = unpack_records(comm.all_gather_rows(packed), cache.record_kind, frame)
    stats = {"rows": rows, "queries": q, "records": len(rec)}
    if len(rec):
        stats["trace"] = train_frame_sharded(cache, rec, comm, steps, batch, ops)
    return (img, img2, term), rows, stats


class ShardedFramePipeline:
    """The sharded frame with rendering and training overlapped (SURVEY.md
    8(e): "render(f) || collect + train(f) ... so the allreduce hides under
    rendering"), the multi-GPU form of frame.FramePipeline:

      frame f:  theta_r <- theta_f                                (render stream)
                render this rank's row band with theta_r, walking this rank's
                share of frame f+1's training paths in the same launch
                all-gather records(f); tile-sharded train(f) with one
                gradient all-reduce per step -> theta_{f+1}         (train stream)

    The walks never read theta, so frame f+1's records collected during
    frame f's launch are the ones run_frame_sharded collects at f+1; each
    frame computes what run_frame_sharded computes, only overlapped.  The
    record all-gather and the gradient all-reduces run on the train stream
    (NCCL orders them after the stream's prior work), so they hide under the
    render of the same frame.  Across an animation boundary the next records
    are collected on their own at the next frame.
    """

    def __init__(self, scene, cache, config, comm, seed, spp=1, train_fraction=0.025, steps=4,
                 batch=None, ops=None):
        self.scene, self.cache, self.config, self.comm = scene, cache, config, comm
        self.seed, self.spp, self.steps, self.batch = seed, spp, steps, batch
        self.train_fraction = train_fraction
        self.ops = ops or DeviceOps()
        self.s_render = torch.cuda.current_stream()
        self.s_train = torch.cuda.Stream()
        self.theta_r = torch.empty_like(cache.theta)
        self.pending = None  # (frame, callable -> this rank's Records of that frame)
        self.train_events = None
        from .frame import ZeroWatch

        self.zero = ZeroWatch(cache)

    def _count(self, scene):
        from .caches import default_train_count

        return default_train_count(scene, self.train_fraction)

    def step(self, frame, out=None):
        """Frame `frame` on this rank: ((img, img2, term) band sums, rows, stats)."""
        from .estimators import render_and_collect, render_device

        cache, comm = self.cache, self.comm
        scene = self.scene = self.scene.at_frame(frame)
        cache.scene = scene
        same_geometry = not any((a.frame <= frame + 1) != (a.frame <= frame)
                                for a in scene.desc.anims)
        h = int(scene.camera[15])
        rows = split_range(h, comm.world, comm.rank)
        count = self._count(scene)
        paths = split_range(count, comm.world, comm.rank)
        if self.pending is not None and self.pending[0] == frame:
            local = self.pending[1]()
            packed = pack_records({k: getattr(local, k) for k, _ in REC_COLS})
        else:
            packed = self.ops.collect_range(scene, cache.seed, frame, paths[0],
                                            paths[1] - paths[0], cache.record_kind)
        self.pending = None
        # theta_f snapshot for the render, after the previous training
        self.s_render.wait_stream(self.s_train)
        self.theta_r.copy_(cache.theta)
        snap = torch.cuda.Event()
        snap.record(self.s_render)
        zero = self.zero.get()
        if same_geometry:
            img, img2, term, q, nxt = render_and_collect(
                scene, self.config, cache, self.seed, self.spp, frame, count=count,
                train_frame=frame + 1, rows=rows, paths=paths, out=out, theta=self.theta_r,
                defer=True, zero=zero)
            self.pending = (frame + 1, nxt)
        else:
            img, img2, term, q = render_device(scene, self.config, cache, self.seed, self.spp,
                                               frame, rows=rows, out=out, theta=self.theta_r,
                                               zero=zero)
        stats = {"rows": rows, "queries": q}
        self.train_events = None
        self.s_train.wait_event(snap)  # theta_f copied; this frame's records complete
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(self.s_train):
            t0.record(self.s_train)
            rec = unpack_records(comm.all_gather_rows(packed), cache.record_kind, frame)
            stats["records"] = len(rec)
            if len(rec):
                stats["trace"] = train_frame_sharded(cache, rec, comm, self.steps, self.batch,
                                                     self.ops)
            t1.record(self.s_train)
            self.zero.after_update(self.s_train)
        self.train_events = (t0, t1)
        return (img, img2, term), rows, stats


def broadcast_cache(cache, comm, src=0):
    """Make every replica equal to rank `src`'s cache state."""
    for t in (cache.theta, cache.adam.m, cache.adam.v, cache.adam._t, cache.adam._skipped):
        comm.broadcast_(t, src)
    return cache


def replicas_identical(cache, comm):
    """True when every rank holds bit-identical θ (max-reduce of the
    difference to rank 0's copy)."""
    ref = cache.theta.clone()
    comm.broadcast_(ref, 0)
    bad = torch.tensor([0 if torch.equal(ref, cache.theta) else 1], dtype=torch.int32,
                       device=cache.theta.device)
    comm.all_reduce_max_(bad)
    return int(bad.item()) == 0


__all__ = ["split_range", "Comm", "DeviceOps", "collect_sharded", "train_frame_sharded",
           "ShardedFramePipeline",
           "render_band", "gather_image", "run_frame_sharded", "broadcast_cache",
           "replicas_identical", "pack_records", "unpack_records", "REC_COLS", "REC_WIDTH"]
