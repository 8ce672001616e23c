"""Generates the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden.py

Every fixture records the reference's own outputs (nirclab 0.1.0) on
seeded inputs; tests compare the oracle and the CUDA path against them.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    import nirclab  # noqa: F401  (fails loudly when the reference is absent)
    from nirclab import rng
    return rng


def measure_queries(n, seed=0):
    """Same recipe as oracle.measure_queries, through the reference's rng."""
    rng = _ref()
    P = rng.P_MEASURE
    pos = rng.uniform_array(seed, P, 0, 3 * n).reshape(n, 3)
    nrm = rng.normal_array(seed, P, 1, 3 * n).reshape(n, 3)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    alb = rng.uniform_array(seed, P, 2, 3 * n).reshape(n, 3)
    rough = rng.uniform_array(seed, P, 3, n)
    dirs = rng.normal_array(seed, P, 4, 3 * n).reshape(n, 3)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return pos, nrm, alb, rough, dirs


def golden_encode():
    """encode_batch + mlp_forward of the default layout, D = 2 and D = 4."""
    from nirclab.encoding import encode_batch
    from nirclab.mlp import init_theta, make_spec, mlp_forward

    n = 4096
    pos, nrm, alb, rough, dirs = measure_queries(n, seed=0)
    out = dict(pos=pos, nrm=nrm, alb=alb, rough=rough, dirs=dirs)
    for depth in (2, 4):
        spec = make_spec(depth=depth)
        theta = init_theta(spec, seed=1, out_scale=0.1)
        X, ent, wts = encode_batch(spec, theta, pos, nrm, alb, rough, dirs)
        Y = mlp_forward(spec, theta, X)
        out[f"Y_d{depth}"] = Y
        if depth == 2:  # the grid draws come first, so X is the same for D=4
            out["X"] = X
            out["entries"] = ent.astype(np.int32)
            out["weights"] = wts
    np.savez_compressed(os.path.join(HERE, "encode_forward.npz"), **out)


def synth_records(n, seed):
    """Deterministic record set (pos in the Cornell box, cosine pdfs)."""
    rng = _ref()
    P = rng.P_MEASURE
    pos = rng.uniform_array(seed, P, 10, 3 * n).reshape(n, 3)
    ns = rng.normal_array(seed, P, 11, 3 * n).reshape(n, 3)
    ns /= np.linalg.norm(ns, axis=1, keepdims=True)
    dirs = rng.normal_array(seed, P, 12, 3 * n).reshape(n, 3)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    cos = np.einsum("ij,ij->i", dirs, ns)
    dirs[cos < 0] *= -1.0
    cos = np.abs(cos)
    pdf = np.maximum(cos, 1e-3) / np.pi
    alb = rng.uniform_array(seed, P, 13, 3 * n).reshape(n, 3)
    rough = np.ones(n)
    target = 3.0 * rng.uniform_array(seed, P, 14, 3 * n).reshape(n, 3) ** 2
    return dict(pos=pos, ns=ns, alb=alb, rough=rough, dirs=dirs, target=target, pdf=pdf)


def golden_train():
    """Two train_frame steps on a small-table net (full theta/m/v kept) for
    n <= cap (permutation) and n > cap (selection)."""
    from nirclab.adam import AdamState
    from nirclab.caches import Records, train_frame
    from nirclab.mlp import init_theta, make_spec

    class _C:  # the attributes train_frame reads from a Cache
        pass

    out = {}
    for tag, n, cap in (("small", 3000, None), ("big", 20000, None)):
        rec = synth_records(n, seed=5)
        spec = make_spec(table=2 ** 12, depth=4, bb_min=np.zeros(3), bb_ext=np.ones(3))
        theta = init_theta(spec, seed=3)
        c = _C()
        c.spec, c.theta, c.adam = spec, theta, AdamState(theta)
        c.seed, c.frame, c.loss_kind, c.loss_eps = 7, 2, "relative_l2", 0.01
        c.running_mean = np.zeros(3)
        c.kind, c.snapshot_dir = "nirc", None
        records = Records(kind="nirc", frame=2, **rec)
        trace = train_frame(c, records, steps=2, batch=cap)
        out[f"{tag}_rec_digest"] = np.array([v.sum() for v in rec.values()])
        out[f"{tag}_trace"] = np.array(trace)
        out[f"{tag}_theta"] = theta
        out[f"{tag}_m"] = c.adam.m
        out[f"{tag}_v"] = c.adam.v
        out[f"{tag}_t"] = np.int64(c.adam.t)
        # the batch idx of each step, straight from the reference's recipe
        from nirclab.rng import P_SHUFFLE, uniform_array
        for s in range(2):
            u = uniform_array(7, P_SHUFFLE, 2, n, offset=s * n)
            out[f"{tag}_idx{s}"] = np.argsort(u, kind="stable")[: min(16384, n)].astype(np.int32)
    np.savez_compressed(os.path.join(HERE, "train_step.npz"), **out)


def golden_losses_adam():
    """Known-answer loss values and 20 Adam steps (incl. a skipped one)."""
    from nirclab.adam import AdamState, adam_step
    from nirclab.losses import loss_l2, loss_relative_l2

    rng = np.random.default_rng(0)
    y = rng.random((64, 3)).astype(np.float32)
    t = rng.random((64, 3))
    pdf = rng.uniform(0.3, 2.0, 64)
    v1, g1 = loss_relative_l2(y, t, pdf)
    v2, g2 = loss_l2(y, t, pdf)
    theta = rng.normal(size=1000).astype(np.float32)
    theta_init = theta.copy()
    st = AdamState(theta)
    grads = rng.normal(size=(20, 1000)).astype(np.float32)
    grads[7, 3] = np.nan
    thetas = []
    for g in grads:
        adam_step(st, theta, g)
        thetas.append(theta.copy())
    np.savez_compressed(os.path.join(HERE, "losses_adam.npz"), y=y, t=t, pdf=pdf,
                        rel_val=v1, rel_grad=g1, l2_val=v2, l2_grad=g2,
                        theta0=theta_init, grads=grads,
                        thetas=np.array(thetas), t_final=st.t, skipped=st.skipped)


if __name__ == "__main__":
    which = sys.argv[1:] or ["encode", "train", "losses"]
    if "encode" in which:
        golden_encode()
    if "train" in which:
        golden_train()
    if "losses" in which:
        golden_losses_adam()
    print("golden fixtures written to", HERE)
