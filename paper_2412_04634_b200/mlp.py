"""Tiny fully connected networks over one flat parameter vector
(drop-in for pkg/src/nirclab/mlp.py).

The parameter layout, ``make_spec`` and ``init_theta`` are host-side and
identical to the reference (same numpy Generator calls, so the same theta
for the same seed).  ``mlp_forward`` / ``mlp_backward`` / ``full_forward``
run on the B200 through the C ABI:

* ``full_forward`` is the fused persistent kernel (encode + tcgen05 3xTF32
  MLP, activations only in SMEM/TMEM) -- the NIRC inference hot path;
* ``mlp_forward`` / ``mlp_backward`` are the fp32 SIMT twin used for the
  reference's batch API and the training step.
"""

from __future__ import annotations

from collections import namedtuple

import numpy as np
import torch

from . import _dev, _lib
from .encoding import AUX_DIM, encode_batch, level_resolutions, scatter_grid_grad
from .errors import DivergenceError

ACT_RELU = 0
ACT_SIGMOID = 1

PRECISION_TF32X3 = 0   # tcgen05.mma kind::tf32, hi/lo split operands
PRECISION_FP32 = 1     # SIMT fp32 twin
PRECISION_F16X2 = 2    # tcgen05.mma kind::f16, fp16 hi/lo split operands

NetSpec = namedtuple(
    "NetSpec",
    ["levels", "table", "feats", "res", "bb_min", "bb_inv", "bands", "in_dim", "nl",
     "w_off", "b_off", "dims", "out_act", "grid_len", "theta_len"],
)


def make_spec(levels=12, table=2 ** 15, feats=2, base_res=4, max_res=256, bands=4,
              depth=4, width=64, out_dim=3, out_act=ACT_RELU, bb_min=None, bb_ext=None):
    """Layout of theta: hash tables, then per layer W (dout x din) and b
    (mlp.py:36-62)."""
    bb_min = np.zeros(3) if bb_min is None else np.asarray(bb_min, float)
    bb_ext = np.ones(3) if bb_ext is None else np.asarray(bb_ext, float)
    in_dim = levels * feats + bands * bands + AUX_DIM
    dims = [in_dim] + [width] * depth + [out_dim]
    grid_len = levels * table * feats
    w_off, b_off = [], []
    cursor = grid_len
    for din, dout in zip(dims[:-1], dims[1:]):
        w_off.append(cursor)
        cursor += din * dout
        b_off.append(cursor)
        cursor += dout
    return NetSpec(levels=levels, table=table, feats=feats,
                   res=level_resolutions(levels, base_res, max_res),
                   bb_min=bb_min, bb_inv=1.0 / bb_ext, bands=bands, in_dim=in_dim,
                   nl=len(dims) - 1, w_off=np.array(w_off, np.int64),
                   b_off=np.array(b_off, np.int64), dims=np.array(dims, np.int64),
                   out_act=out_act, grid_len=grid_len, theta_len=cursor)


def init_theta(spec, seed=0, dtype=np.float32, out_scale=0.0):
    """Uniform(+-1e-4) grid, He-normal hidden layers, zero biases, zero (or
    N(0, out_scale)) output layer -- the same Generator draws as
    mlp.py:65-85."""
    gen = np.random.default_rng(seed)
    theta = np.zeros(spec.theta_len, dtype)
    theta[: spec.grid_len] = gen.uniform(-1e-4, 1e-4, spec.grid_len)
    for layer in range(spec.nl):
        din = int(spec.dims[layer])
        dout = int(spec.dims[layer + 1])
        w = int(spec.w_off[layer])
        if layer == spec.nl - 1:
            if out_scale > 0.0:
                theta[w: w + din * dout] = gen.normal(0.0, out_scale, din * dout)
        else:
            theta[w: w + din * dout] = gen.normal(0.0, np.sqrt(2.0 / din), din * dout)
    return theta


def weight_view(spec, theta, layer):
    w = int(spec.w_off[layer])
    din = int(spec.dims[layer])
    dout = int(spec.dims[layer + 1])
    return theta[w: w + din * dout].reshape(dout, din)


def bias_view(spec, theta, layer):
    b = int(spec.b_off[layer])
    return theta[b: b + int(spec.dims[layer + 1])]


def _zs_width(spec):
    return int(sum(int(d) for d in spec.dims[1:]))


def _mlp_forward_f64(spec, theta, X, training):
    host = _dev.is_host(X)
    th = _dev.dev(theta, torch.float64)
    x = _dev.dev(X, torch.float64)
    if x.dim() == 1:
        x = x.reshape(1, -1)
    n = int(x.shape[0])
    Y = _dev.empty((n, int(spec.dims[-1])), torch.float64)
    zs = _dev.empty((n, _zs_width(spec)), torch.float64) if training else None
    flag = _dev.zeros((1,), torch.int32)
    lib = _lib.load()
    _lib.check(lib.nirc_mlp_forward_f64(_lib.make_c_spec(spec), _dev.ptr(th), _dev.ptr(x), n,
                                        _dev.ptr(Y), _dev.ptr(zs), _dev.ptr(flag),
                                        _dev.stream()), "nirc_mlp_forward_f64")
    if int(flag.item()) != 0:
        raise DivergenceError("non-finite network parameter")
    if training:
        return _dev.out(Y, host), (x, zs)
    return _dev.out(Y, host)


def mlp_forward(spec, theta, X, training=False):
    """Batch forward (mlp.py:102-122).  Returns Y, or (Y, cache) when
    training; the cache holds X and every pre-activation for mlp_backward.
    Raises DivergenceError if theta holds a non-finite value.  A float64
    theta runs the reference's 64-bit shadow mode (fp64 kernels)."""
    if _dev.is_f64(theta):
        return _mlp_forward_f64(spec, theta, X, training)
    host = _dev.is_host(X)
    th = _dev.dev(theta, torch.float32)
    x = _dev.dev(X, torch.float32)
    if x.dim() == 1:
        x = x.reshape(1, -1)
    n = int(x.shape[0])
    dout = int(spec.dims[-1])
    Y = _dev.empty((n, dout), torch.float32)
    zs = _dev.empty((n, _zs_width(spec)), torch.float32) if training else None
    flag = _dev.zeros((1,), torch.int32)
    lib = _lib.load()
    _lib.check(lib.nirc_mlp_forward(_lib.make_c_spec(spec), _dev.ptr(th), _dev.ptr(x), n,
                                    _dev.ptr(Y), _dev.ptr(zs), _dev.ptr(flag), _dev.stream()),
               "nirc_mlp_forward")
    if int(flag.item()) != 0:
        raise DivergenceError("non-finite network parameter")
    if training:
        return _dev.out(Y, host), (x, zs)
    return _dev.out(Y, host)


def _mlp_backward_f64(spec, theta, cache, dY, entries, weights):
    X, zs = cache
    host = _dev.is_host(dY)
    th = _dev.dev(theta, torch.float64)
    dy = _dev.dev(dY, torch.float64)
    n = int(X.shape[0])
    g = _dev.zeros((spec.theta_len,), torch.float64)
    dX = _dev.empty((n, spec.in_dim), torch.float64)
    scratch = _dev.empty((n, _zs_width(spec)), torch.float64)
    lib = _lib.load()
    _lib.check(lib.nirc_mlp_backward_f64(_lib.make_c_spec(spec), _dev.ptr(th), _dev.ptr(X),
                                         _dev.ptr(zs), _dev.ptr(dy), n, _dev.ptr(g),
                                         _dev.ptr(dX), _dev.ptr(scratch), _dev.stream()),
               "nirc_mlp_backward_f64")
    if entries is not None:
        scatter_grid_grad(spec, g, _dev.dev(entries, torch.int64),
                          _dev.dev(weights, torch.float32), dX)
    return _dev.out(g, host)


def mlp_backward(spec, theta, cache, dY, entries=None, weights=None):
    """Reverse mode (mlp.py:125-154); ReLU' is (z >= 0) on every layer.
    Returns a gradient congruent to theta (float64 in the shadow mode)."""
    if _dev.is_f64(theta):
        return _mlp_backward_f64(spec, theta, cache, dY, entries, weights)
    X, zs = cache
    host = _dev.is_host(dY)
    th = _dev.dev(theta, torch.float32)
    dy = _dev.dev(dY, torch.float32)
    n = int(X.shape[0])
    g = _dev.zeros((spec.theta_len,), torch.float32)
    dX = _dev.empty((n, spec.in_dim), torch.float32)
    scratch = _dev.empty((n, _zs_width(spec)), torch.float32)
    lib = _lib.load()
    _lib.check(lib.nirc_mlp_backward(_lib.make_c_spec(spec), _dev.ptr(th), _dev.ptr(X),
                                     _dev.ptr(zs), _dev.ptr(dy), n, _dev.ptr(g), _dev.ptr(dX),
                                     _dev.ptr(scratch), _dev.stream()),
               "nirc_mlp_backward")
    if entries is not None:
        scatter_grid_grad(spec, g, _dev.dev(entries, torch.int64),
                          _dev.dev(weights, torch.float32), dX)
    return _dev.out(g, host)


_PIPE = {}


def _pipe_streams():
    dev = torch.cuda.current_device()
    st = _PIPE.get(dev)
    if st is None:
        st = (torch.cuda.Stream(), torch.cuda.Stream())
        _PIPE[dev] = st
    return st


def _pinned_host(arrays):
    return all(isinstance(a, torch.Tensor) and not a.is_cuda and a.is_pinned() for a in arrays)


_PIPE_CHUNK = int(__import__("os").environ.get("NIRC_PIPE_CHUNK", 1 << 18))  # measured: 2^18 best of 2^17..2^20


def _full_forward_pipelined(spec, th, host, precision, out=None, chunk=None):
    """Host-resident (pinned) query rows: chunked H2D copies on one stream,
    the fused kernel on the caller's stream, D2H of the outputs on a third,
    double-buffered so PCIe transfers in both directions overlap the compute.
    Returns a pinned host tensor; the caller's stream is ordered after it."""
    n = int(host[0].shape[0])
    dout = int(spec.dims[-1])
    if chunk is None:
        chunk = _PIPE_CHUNK
    cur = torch.cuda.current_stream()
    s_in, s_out = _pipe_streams()
    y_host = out if out is not None else torch.empty((n, dout), dtype=torch.float32,
                                                     pin_memory=True)
    widths = [3, 3, 3, 1, 3]
    m = min(chunk, n)
    bufs = [[_dev.empty((m, w) if w > 1 else (m,), torch.float64) for w in widths]
            for _ in range(2)]
    ybuf = [_dev.empty((m, dout), torch.float32) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    lib = _lib.load()
    cs = _lib.make_c_spec(spec)
    flags = _dev.zeros((1,), torch.int32)
    s_in.wait_stream(cur)
    for k, lo in enumerate(range(0, n, m)):
        hi = min(n, lo + m)
        b = k % 2
        with torch.cuda.stream(s_in):
            if k >= 2:
                s_in.wait_event(ev_comp[b])  # the kernel of chunk k-2 read bufs[b]
            for d, h in zip(bufs[b], host):
                d[: hi - lo].copy_(h[lo:hi], non_blocking=True)
            ev_in[b].record(s_in)
        cur.wait_event(ev_in[b])
        if k >= 2:
            cur.wait_event(ev_out[b])  # chunk k-2's outputs left ybuf[b]
        st = lib.nirc_full_forward(cs, _dev.ptr(th), *[_dev.ptr(d) for d in bufs[b]], hi - lo,
                                   _dev.ptr(ybuf[b]), int(precision),
                                   _dev.ptr(flags) if k == 0 else _dev.ptr(None), _dev.stream())
        _lib.check(st, "nirc_full_forward")
        ev_comp[b].record(cur)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_comp[b])
            y_host[lo:hi].copy_(ybuf[b][: hi - lo], non_blocking=True)
            ev_out[b].record(s_out)
    for b in range(2):
        for d in bufs[b]:
            d.record_stream(s_in)
        ybuf[b].record_stream(s_out)
    cur.wait_stream(s_out)
    # the host result is complete only when the last D2H copy has landed:
    # wait for it before handing the buffer to the caller (and raise the
    # reference's DivergenceError on a non-finite theta, mlp.py:104-105)
    s_out.synchronize()
    _lib.check_flags(flags, "full_forward")
    return y_host


_NP_STAGING = {}


def _np_staging(m, dout):
    """Two pinned staging sets (5 input columns + outputs) of m rows, reused."""
    key = (m, dout)
    st = _NP_STAGING.get(key)
    if st is None:
        widths = [3, 3, 3, 1, 3]
        inp = [[torch.empty((m, w) if w > 1 else (m,), dtype=torch.float64, pin_memory=True)
                for w in widths] for _ in range(2)]
        ys = [torch.empty((m, dout), dtype=torch.float32, pin_memory=True) for _ in range(2)]
        st = (inp, ys)
        _NP_STAGING[key] = st
    return st


def _full_forward_numpy(spec, th, rows, precision, chunk=None):
    """numpy (pageable) query rows, the reference's types: each chunk is
    copied into a pinned staging buffer on the host (multi-threaded torch
    copy) while the previous chunk's H2D copy, kernel and D2H copy run; the
    outputs drain from pinned staging into the numpy result the same way.
    Returns a fresh numpy (n, dout) f32 array."""
    n = int(rows[0].shape[0])
    dout = int(spec.dims[-1])
    m = min(chunk or _PIPE_CHUNK, n)
    inp, ys = _np_staging(m, dout)
    y = np.empty((n, dout), np.float32)
    cur = torch.cuda.current_stream()
    s_in, s_out = _pipe_streams()
    widths = [3, 3, 3, 1, 3]
    dbuf = [[_dev.empty((m, w) if w > 1 else (m,), torch.float64) for w in widths]
            for _ in range(2)]
    ybuf = [_dev.empty((m, dout), torch.float32) for _ in range(2)]
    ev_h2d = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_d2h = [torch.cuda.Event() for _ in range(2)]
    lib = _lib.load()
    cs = _lib.make_c_spec(spec)
    flags = _dev.zeros((1,), torch.int32)
    s_in.wait_stream(cur)
    pending = None  # (buffer, lo, hi) of the chunk whose outputs drain next
    for k, lo in enumerate(range(0, n, m)):
        hi = min(n, lo + m)
        c = hi - lo
        b = k % 2
        if k >= 2:
            ev_h2d[b].synchronize()  # the H2D copy of chunk k-2 has read staging b
        for t, a in zip(inp[b], rows):
            t[:c].copy_(torch.from_numpy(a[lo:hi]))
        with torch.cuda.stream(s_in):
            if k >= 2:
                s_in.wait_event(ev_comp[b])  # the kernel of chunk k-2 read dbuf[b]
            for d, t in zip(dbuf[b], inp[b]):
                d[:c].copy_(t[:c], non_blocking=True)
            ev_h2d[b].record(s_in)
        cur.wait_event(ev_h2d[b])
        if k >= 2:
            cur.wait_event(ev_d2h[b])  # chunk k-2's outputs left ybuf[b]
        st = lib.nirc_full_forward(cs, _dev.ptr(th), *[_dev.ptr(d) for d in dbuf[b]], c,
                                   _dev.ptr(ybuf[b]), int(precision),
                                   _dev.ptr(flags) if k == 0 else _dev.ptr(None), _dev.stream())
        _lib.check(st, "nirc_full_forward")
        ev_comp[b].record(cur)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_comp[b])
            ys[b][:c].copy_(ybuf[b][:c], non_blocking=True)
            ev_d2h[b].record(s_out)
        if pending is not None:  # drain the previous chunk while this one runs
            pb, plo, phi = pending
            ev_d2h[pb].synchronize()
            y[plo:phi] = ys[pb][: phi - plo].numpy()
        pending = (b, lo, hi)
    pb, plo, phi = pending
    ev_d2h[pb].synchronize()
    y[plo:phi] = ys[pb][: phi - plo].numpy()
    for b in range(2):
        for d in dbuf[b]:
            d.record_stream(s_in)
        ybuf[b].record_stream(s_out)
    cur.wait_stream(s_out)
    _lib.check_flags(flags, "full_forward")
    return y


def query(spec, theta, surf, dirs, dir_to_surf, precision=PRECISION_F16X2):
    """Directions against shared surfaces (Cache._query, caches.py:211-233,
    batched): surf (n_s, 10) rows pos.xyz | ns.xyz | albedo.rgb | roughness,
    dirs (n, 3), dir_to_surf (n,) -> (n, dout) f32, through the C ABI's
    nirc_query (surface rows gathered on the device, fused encode + MLP).
    numpy in -> numpy out; CUDA tensors stay on the device."""
    host = _dev.is_host(dirs)
    th = _dev.dev(theta, torch.float32)
    S = _dev.dev(surf, torch.float64)
    D = _dev.dev(dirs, torch.float64)
    idx = _dev.dev(dir_to_surf, torch.int32)
    n = int(D.shape[0])
    Y = _dev.empty((n, int(spec.dims[-1])), torch.float32)
    if n:
        lib = _lib.load()
        flags = _dev.zeros((1,), torch.int32)
        st = lib.nirc_query(_lib.make_c_spec(spec), _dev.ptr(th), _dev.ptr(S), int(S.shape[0]),
                            _dev.ptr(D), _dev.ptr(idx), n, _dev.ptr(Y), int(precision),
                            _dev.ptr(flags), _dev.stream())
        if st == _lib.NIRC_E_UNSUPPORTED:  # non-default layouts: generic device path
            il = idx.long()
            if int(il.min()) < 0 or int(il.max()) >= int(S.shape[0]):
                raise _lib.ConfigError("nirc_query: dir_to_surf index outside [0, n_surf)")
            Y = full_forward(spec, th, S[il, 0:3], S[il, 3:6], S[il, 6:9], S[il, 9], D,
                             precision=precision)
        else:
            _lib.check(st, "nirc_query")
            _lib.check_flags(flags, "nirc_query")
    return Y.cpu().numpy() if host else Y


def full_forward(spec, theta, pos, normal, albedo, rough, dirs, training=False,
                 precision=PRECISION_F16X2, out=None):
    """encode_batch + mlp_forward (mlp.py:216-224).  Inference runs the fused
    tcgen05 kernel (2xFP16 split by default; precision 0 = 3xTF32, 1 = fp32
    SIMT twin); pinned host tensors stream through a copy/compute/copy
    pipeline (into `out`, a pinned (n, 3) f32 tensor, when given); training
    returns the reference tuple via the SIMT path."""
    if training or _dev.is_f64(theta):  # the batch pipeline (and the f64 shadow mode)
        X, entries, weights = encode_batch(spec, theta, pos, normal, albedo, rough, dirs)
        if not training:
            return mlp_forward(spec, theta, X)
        Y, cache = mlp_forward(spec, theta, X, training=True)
        return Y, cache, entries, weights
    host = _dev.is_host(pos)
    th = _dev.dev(theta, torch.float32)
    rows = (pos, normal, albedo, rough, dirs)
    if (_pinned_host(rows) and all(r.dtype == torch.float64 for r in rows)
            and int(pos.shape[0]) > 0):
        from .encoding import is_default_layout

        if is_default_layout(spec):
            return _full_forward_pipelined(spec, th, [r.contiguous() for r in rows], precision,
                                           out)
    if (out is None and all(isinstance(r, np.ndarray) and r.dtype == np.float64 for r in rows)
            and int(pos.shape[0]) >= (1 << 18)):
        from .encoding import is_default_layout

        if is_default_layout(spec):  # large numpy batches: staged, overlapped copies
            return _full_forward_numpy(spec, th, [np.ascontiguousarray(r) for r in rows],
                                       precision)
    args = [_dev.dev(a, torch.float64) for a in rows]
    n = int(args[0].shape[0])
    Y = _dev.empty((n, int(spec.dims[-1])), torch.float32)
    lib = _lib.load()
    flags = _dev.zeros((1,), torch.int32)
    st = lib.nirc_full_forward(_lib.make_c_spec(spec), _dev.ptr(th),
                               *[_dev.ptr(a) for a in args], n, _dev.ptr(Y), int(precision),
                               _dev.ptr(flags), _dev.stream())
    if st == _lib.NIRC_E_UNSUPPORTED:
        # non-default layouts (tests' tiny nets) take the generic device path
        X, _, _ = encode_batch(spec, th, *args)
        return _dev.out(mlp_forward(spec, th, X), host)
    _lib.check(st, "nirc_full_forward")
    # mlp.py:104-105: a non-finite theta raises DivergenceError (reads the
    # device flag, i.e. waits for the launch)
    _lib.check_flags(flags, "full_forward")
    return _dev.out(Y, host)


def mlp_forward_s(spec, theta, xin, h1=None, h2=None):
    """Scalar forward of one encoded input (mlp.py:160-192): the first three
    outputs as a tuple (unused slots zero).  h1/h2 (the reference's scratch
    rows) are accepted and unused: the device kernel keeps its own."""
    X = np.asarray(xin, np.float32).reshape(1, -1)
    Y = mlp_forward(spec, theta, X)
    y = np.asarray(Y, np.float64).reshape(-1)
    out = [float(y[i]) if i < y.size else 0.0 for i in range(3)]
    return out[0], out[1], out[2]


def forward_scalar_reference(spec, theta, xin):
    """Naive per-neuron forward of one encoded input, the reference's test
    oracle (mlp.py:195-213): python-float (f64) sums in (bias, i ascending)
    order.  Host code by design -- it is the checker, not a kernel."""
    theta = np.asarray(theta.cpu() if isinstance(theta, torch.Tensor) else theta)
    cur = [float(v) for v in np.asarray(xin).ravel()]
    for layer in range(spec.nl):
        din = int(spec.dims[layer])
        dout = int(spec.dims[layer + 1])
        w = int(spec.w_off[layer])
        b = int(spec.b_off[layer])
        nxt = []
        for j in range(dout):
            acc = float(theta[b + j])
            for i in range(din):
                acc += cur[i] * float(theta[w + j * din + i])
            if layer < spec.nl - 1 or spec.out_act == ACT_RELU:
                nxt.append(max(acc, 0.0))
            else:
                nxt.append(1.0 / (1.0 + np.exp(-acc)))
        cur = nxt
    return np.array(cur)


def gradient_check(spec, theta, surf, target, pdf, loss_kind="l2", h=1e-3, eps=0.01,
                   running_mean=None, indices=None):
    """Five-point central-difference check of the full reverse-mode gradient
    (mlp.py:227-292): the device forward / losses / backward (+ grid
    scatter) against finite differences of the device loss, in theta's
    dtype (float64 = the shadow mode, where the 1e-5 bar is meaningful).
    The relative-L2 denominator and the variance running mean are frozen
    across the perturbed evaluations.  Returns the maximum relative error
    over the checked indices (default: every parameter)."""
    from . import losses

    pos, normal, albedo, rough, dirs = surf
    theta = np.asarray(theta)
    if running_mean is None:
        running_mean = np.array([0.3, 0.2, 0.1])
    Y0, cache, entries, weights = full_forward(spec, theta, pos, normal, albedo, rough, dirs,
                                               training=True)
    frozen = losses.relative_l2_denom(np.asarray(Y0), eps)

    def eval_loss(th, want_grad=False):
        if want_grad:
            Y, cc, en, we = full_forward(spec, th, pos, normal, albedo, rough, dirs,
                                         training=True)
        else:
            Y = full_forward(spec, th, pos, normal, albedo, rough, dirs)
        Y = np.asarray(Y)
        if loss_kind == "l2":
            val, dY = losses.loss_l2(Y, target, pdf)
        elif loss_kind == "relative_l2":
            val, dY = losses.loss_relative_l2(Y, target, pdf, eps, frozen_denom=frozen)
        elif loss_kind == "variance":
            val, dY = losses.loss_variance(Y, target, pdf, running_mean)
        elif loss_kind == "bce":
            val, dY = losses.loss_bce(Y, target)
        else:
            raise ValueError(loss_kind)
        if want_grad:
            return val, np.asarray(mlp_backward(spec, th, cc, dY, en, we))
        return val

    _, g = eval_loss(theta, want_grad=True)
    if indices is None:
        indices = range(spec.theta_len)
    gscale = np.abs(g).max()
    worst = 0.0
    for i in indices:
        keep = theta[i]
        vals = []
        for step in (h, -h, 2.0 * h, -2.0 * h):
            theta[i] = keep + step
            vals.append(eval_loss(theta))
        theta[i] = keep
        up, dn, up2, dn2 = vals
        fd = (8.0 * (up - dn) - (up2 - dn2)) / (12.0 * h)
        denom = max(abs(fd), abs(g[i]), 1e-4 * gscale, 1e-12)
        worst = max(worst, abs(fd - g[i]) / denom)
    return worst
