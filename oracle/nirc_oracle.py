"""CPU ORACLE for the NIRC hot path -- TEST INFRASTRUCTURE ONLY.

A plain-numpy restatement of the reference algorithm (``nirclab`` 0.1.0,
pkg/src/nirclab/*.py), used as the checker by tests/, by
``__graft_entry__.smoke()`` and as ``bench.py``'s CPU baseline leg.  The
product path (``paper_2412_04634_b200``) never imports this module.

Each function cites the reference lines it restates.  The oracle is pinned
against golden vectors produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz;
tests/test_oracle_golden.py).
"""

from __future__ import annotations

import math

import numpy as np

# ------------------------------------------------------------------ rng --
# pkg/src/nirclab/rng.py:23-31, 59-106
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1
P_RENDER, P_TRAIN, P_INIT, P_SHUFFLE, P_BASELINE, P_MEASURE = 1, 2, 3, 4, 5, 6


def mix64_int(x):
    x = (int(x) + 0x9E3779B97F4A7C15) & _MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK
    return x ^ (x >> 31)


def stream_key(seed, purpose, frame, pixel, sample):
    k = mix64_int(int(seed) ^ int(purpose))
    k = mix64_int(k ^ int(frame))
    k = mix64_int(k ^ int(pixel))
    return mix64_int(k ^ int(sample))


def _mix64_vec(x):
    with np.errstate(over="ignore"):
        x = x + _G
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        return x ^ (x >> np.uint64(31))


def uniform_bits(seed, purpose, stream, count, offset=0):
    """(u64 draw) >> 11 for dims offset..offset+count (rng.py:100-106)."""
    key = np.uint64(stream_key(seed, purpose, 0, stream, 0))
    dims = np.arange(offset, offset + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix64_vec(key + _G * dims) >> np.uint64(11)


def uniform_array(seed, purpose, stream, count, offset=0):
    return uniform_bits(seed, purpose, stream, count, offset).astype(np.float64) \
        * (1.0 / 9007199254740992.0)


def normal_array(seed, purpose, stream, count, offset=0):
    """Box-Muller on addressed draws (rng.py:109-119)."""
    h = (count + 1) // 2
    u = uniform_array(seed, purpose, stream, 2 * h, offset)
    r = np.sqrt(-2.0 * np.log(np.clip(u[:h], 1e-16, 1.0)))
    z = np.empty(2 * h)
    z[:h] = r * np.cos(2.0 * np.pi * u[h:])
    z[h:] = r * np.sin(2.0 * np.pi * u[h:])
    return z[:count]


# ------------------------------------------------------------------- SH --
# pkg/src/nirclab/sh.py:21-33 (normalisation), :89-127 (batch evaluation)
def _norm(l, m):
    return math.sqrt((2 * l + 1) / (4.0 * math.pi) * math.factorial(l - m)
                     / math.factorial(l + m))


def sh_batch(d, bands):
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    s = np.sqrt(x * x + y * y)
    ok = s > 0.0
    safe = np.where(ok, s, 1.0)
    cphi = np.where(ok, x / safe, 1.0)
    sphi = np.where(ok, y / safe, 0.0)
    out = np.empty((d.shape[0], bands * bands))
    cm, sm, pmm = np.ones_like(z), np.zeros_like(z), np.ones_like(z)
    for m in range(bands):
        if m > 0:
            pmm = pmm * (2.0 * m - 1.0) * s
            cm, sm = cm * cphi - sm * sphi, sm * cphi + cm * sphi
        p2 = np.zeros_like(z)
        p1 = np.zeros_like(z)
        for l in range(m, bands):
            if l == m:
                p = pmm
            elif l == m + 1:
                p = z * (2.0 * m + 1.0) * pmm
            else:
                p = ((2.0 * l - 1.0) * z * p1 - (l + m - 1.0) * p2) / (l - m)
            p2, p1 = p1, p
            c = l * l + l
            if m == 0:
                out[:, c] = _norm(l, 0) * p
            else:
                k = math.sqrt(2.0) * _norm(l, m)
                out[:, c + m] = k * p * cm
                out[:, c - m] = k * p * sm
    return out


# ------------------------------------------------------------- network ---
class Spec:
    """Plain restatement of NetSpec/make_spec (mlp.py:26-62)."""

    def __init__(self, levels=12, table=2 ** 15, feats=2, base_res=4, max_res=256,
                 bands=4, depth=4, width=64, out_dim=3, out_act=0, bb_min=None,
                 bb_ext=None):
        self.levels, self.table, self.feats, self.bands = levels, table, feats, bands
        self.out_act = out_act
        if levels == 1:
            self.res = np.array([base_res], np.int64)
        else:
            b = np.exp(np.log(max_res / base_res) / (levels - 1))
            self.res = np.floor(base_res * b ** np.arange(levels) + 0.5).astype(np.int64)
        self.bb_min = np.zeros(3) if bb_min is None else np.asarray(bb_min, float)
        self.bb_inv = 1.0 / (np.ones(3) if bb_ext is None else np.asarray(bb_ext, float))
        self.in_dim = levels * feats + bands * bands + 7
        self.dims = [self.in_dim] + [width] * depth + [out_dim]
        self.nl = len(self.dims) - 1
        self.grid_len = levels * table * feats
        self.w_off, self.b_off = [], []
        off = self.grid_len
        for a, b_ in zip(self.dims[:-1], self.dims[1:]):
            self.w_off.append(off)
            off += a * b_
            self.b_off.append(off)
            off += b_
        self.theta_len = off

    def W(self, theta, l):
        return theta[self.w_off[l]: self.w_off[l] + self.dims[l] * self.dims[l + 1]].reshape(
            self.dims[l + 1], self.dims[l])

    def b(self, theta, l):
        return theta[self.b_off[l]: self.b_off[l] + self.dims[l + 1]]


def init_theta(spec, seed=0, out_scale=0.0):
    """mlp.py:65-85 (same Generator call sequence)."""
    rng = np.random.default_rng(seed)
    th = np.zeros(spec.theta_len, np.float32)
    th[: spec.grid_len] = rng.uniform(-1e-4, 1e-4, spec.grid_len)
    for l in range(spec.nl):
        din, dout = spec.dims[l], spec.dims[l + 1]
        w = spec.w_off[l]
        if l == spec.nl - 1:
            if out_scale > 0.0:
                th[w: w + din * dout] = rng.normal(0.0, out_scale, din * dout)
        else:
            th[w: w + din * dout] = rng.normal(0.0, np.sqrt(2.0 / din), din * dout)
    return th


_P1, _P2 = np.uint64(2654435761), np.uint64(805459861)


def encode_batch(spec, theta, pos, normal, albedo, rough, dirs):
    """encoding.py:111-157: returns X (f32), entries (i64), weights (f32)."""
    B, L, F = pos.shape[0], spec.levels, spec.feats
    S = spec.bands ** 2
    X = np.zeros((B, spec.in_dim), np.float32)
    u = np.clip((pos - spec.bb_min[None]) * spec.bb_inv[None], 0.0, 1.0).astype(np.float32)
    ent = np.empty((B, L, 8), np.int64)
    wts = np.empty((B, L, 8), np.float32)
    grid = theta[: spec.grid_len].reshape(L * spec.table, F)
    for lvl in range(L):
        s = (u * np.float32(spec.res[lvl])).astype(np.float32)
        i0 = np.floor(s).astype(np.int64)
        fr = s - i0.astype(np.float32)
        for c in range(8):
            off = np.array([c & 1, (c >> 1) & 1, (c >> 2) & 1], np.int64)
            idx = (i0 + off[None]).astype(np.uint64)
            with np.errstate(over="ignore"):
                h = (idx[:, 0] ^ (idx[:, 1] * _P1) ^ (idx[:, 2] * _P2)) & np.uint64(spec.table - 1)
            w = np.ones(B, np.float32)
            for ax in range(3):
                w = w * (fr[:, ax] if off[ax] else np.float32(1.0) - fr[:, ax])
            slot = lvl * spec.table + h.astype(np.int64)
            ent[:, lvl, c] = slot
            wts[:, lvl, c] = w
            X[:, lvl * F:(lvl + 1) * F] += w[:, None] * grid[slot]
    X[:, L * F: L * F + S] = sh_batch(dirs, spec.bands).astype(np.float32)
    a0 = L * F + S
    X[:, a0: a0 + 3] = ((normal + 1.0) * 0.5).astype(np.float32)
    X[:, a0 + 3: a0 + 6] = albedo.astype(np.float32)
    X[:, a0 + 6] = rough.astype(np.float32)
    return X, ent, wts


def mlp_forward(spec, theta, X, training=False):
    """mlp.py:102-122 in f32 (numpy matmul)."""
    a = X
    acts, zs = [X], []
    for l in range(spec.nl):
        z = a @ spec.W(theta, l).T + spec.b(theta, l)
        if l < spec.nl - 1 or spec.out_act == 0:
            a = np.maximum(z, 0.0)
        else:
            a = 1.0 / (1.0 + np.exp(-z))
        zs.append(z)
        if l < spec.nl - 1:
            acts.append(a)
    return (a, (acts, zs)) if training else a


def mlp_backward(spec, theta, cache, dY, entries, weights):
    """mlp.py:125-154 + encoding.py:160-167."""
    acts, zs = cache
    g = np.zeros_like(theta)
    zo = zs[-1]
    if spec.out_act == 0:
        dz = dY * (zo >= 0.0)
    else:
        s = 1.0 / (1.0 + np.exp(-zo))
        dz = dY * s * (1.0 - s)
    dX = None
    for l in range(spec.nl - 1, -1, -1):
        spec.W(g, l)[...] += dz.T @ acts[l]
        spec.b(g, l)[...] += dz.sum(axis=0)
        da = dz @ spec.W(theta, l)
        if l > 0:
            dz = da * (zs[l - 1] >= 0.0)
        else:
            dX = da
    F, L = spec.feats, spec.levels
    dG = dX[:, : L * F].reshape(dX.shape[0], L, F)
    for f in range(F):
        np.add.at(g, entries * F + f, weights * dG[:, :, f][:, :, None])
    return g


def loss_relative_l2(y, t, pdf, eps=0.01):
    """losses.py:33-42 (denominator f32 by numpy promotion)."""
    den = y * y + np.float32(eps)
    p = pdf[:, None]
    diff = y - t
    val = diff * diff / (p * den)
    return float(val.mean()), 2.0 * diff / (p * den) / val.size


def loss_l2(y, t, pdf):
    """losses.py:23-30."""
    p = pdf[:, None]
    diff = y - t
    val = diff * diff / p
    return float(val.mean()), 2.0 * diff / p / val.size


class Adam:
    """adam.py:8-33 in f32."""

    def __init__(self, n, lr=0.01, b1=0.9, b2=0.99, eps=1e-8):
        self.m = np.zeros(n, np.float32)
        self.v = np.zeros(n, np.float32)
        self.t = 0
        self.skipped = 0
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps

    def step(self, theta, g):
        if not np.all(np.isfinite(g)):
            self.skipped += 1
            return False
        self.t += 1
        self.m += np.float32(1.0 - self.b1) * (g - self.m)
        self.v += np.float32(1.0 - self.b2) * (g * g - self.v)
        mh = self.m / np.float32(1.0 - self.b1 ** self.t)
        vh = self.v / np.float32(1.0 - self.b2 ** self.t)
        theta -= (np.float32(self.lr) * mh / (np.sqrt(vh) + np.float32(self.eps))).astype(
            np.float32)
        return True


def select_batch(seed, frame, step, n, cap=16384):
    """caches.py:327-329: stable argsort of the shuffle stream."""
    bits = uniform_bits(seed, P_SHUFFLE, frame, n, offset=step * n)
    return np.argsort(bits, kind="stable")[: min(cap, n)]


def train_step(spec, theta, adam, rec, seed, frame, step, cap=16384, loss="relative_l2"):
    """One optimizer step of train_frame (caches.py:310-354)."""
    n = rec["pos"].shape[0]
    idx = select_batch(seed, frame, step, n, cap)
    X, ent, wts = encode_batch(spec, theta, rec["pos"][idx], rec["ns"][idx], rec["alb"][idx],
                               rec["rough"][idx], rec["dirs"][idx])
    y, cache = mlp_forward(spec, theta, X, training=True)
    if loss == "l2":
        val, dy = loss_l2(y, rec["target"][idx], rec["pdf"][idx])
    else:
        val, dy = loss_relative_l2(y, rec["target"][idx], rec["pdf"][idx])
    g = mlp_backward(spec, theta, cache, dy.astype(np.float32), ent, wts)
    adam.step(theta, g)
    return val, idx


def full_forward(spec, theta, pos, normal, albedo, rough, dirs):
    X, _, _ = encode_batch(spec, theta, pos, normal, albedo, rough, dirs)
    return mlp_forward(spec, theta, X)


# ------------------------------------------------------------ workloads --
def measure_queries(n, seed=0):
    """BASELINE config 2 query recipe: columns drawn from
    the P_MEASURE streams 0..4; pos in [0,1)^3, unit normals and directions
    from normalised normal_array triples, albedo U[0,1)^3, rough U[0,1)."""
    pos = uniform_array(seed, P_MEASURE, 0, 3 * n).reshape(n, 3)
    nrm = normal_array(seed, P_MEASURE, 1, 3 * n).reshape(n, 3)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    alb = uniform_array(seed, P_MEASURE, 2, 3 * n).reshape(n, 3)
    rough = uniform_array(seed, P_MEASURE, 3, n)
    dirs = normal_array(seed, P_MEASURE, 4, 3 * n).reshape(n, 3)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return pos, nrm, alb, rough, dirs


def synth_records(n, seed):
    """Deterministic training-record set used by the train-step fixtures
    (tests/golden/make_golden.py:synth_records, same P_MEASURE streams)."""
    pos = uniform_array(seed, P_MEASURE, 10, 3 * n).reshape(n, 3)
    ns = normal_array(seed, P_MEASURE, 11, 3 * n).reshape(n, 3)
    ns /= np.linalg.norm(ns, axis=1, keepdims=True)
    dirs = normal_array(seed, P_MEASURE, 12, 3 * n).reshape(n, 3)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    cos = np.einsum("ij,ij->i", dirs, ns)
    dirs[cos < 0] *= -1.0
    pdf = np.maximum(np.abs(cos), 1e-3) / np.pi
    alb = uniform_array(seed, P_MEASURE, 13, 3 * n).reshape(n, 3)
    rough = np.ones(n)
    target = 3.0 * uniform_array(seed, P_MEASURE, 14, 3 * n).reshape(n, 3) ** 2
    return dict(pos=pos, ns=ns, alb=alb, rough=rough, dirs=dirs, target=target, pdf=pdf)
