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


def golden_train1():
    """ONE train_frame step per record set (m starts at 0, so the Adam
    moment m = f32(0.1) * g and v = f32(0.01) * g^2 expose the reference's
    raw gradient of the step: mlp_backward + scatter_grid_grad)."""
    from nirclab.adam import AdamState
    from nirclab.caches import Records, train_frame
    from nirclab.mlp import init_theta, make_spec

    class _C:
        pass

    out = {}
    for tag, n in (("small", 3000), ("big", 20000)):
        rec = synth_records(n, seed=5)
        spec = make_spec(table=2 ** 12, depth=4, bb_min=np.zeros(3), bb_ext=np.ones(3))
        theta = init_theta(spec, seed=3, out_scale=0.05)
        c = _C()
        c.spec, c.theta, c.adam = spec, theta, AdamState(theta)
        c.seed, c.frame, c.loss_kind, c.loss_eps = 7, 2, "relative_l2", 0.01
        c.running_mean = np.zeros(3)
        c.kind, c.snapshot_dir = "nirc", None
        trace = train_frame(c, Records(kind="nirc", frame=2, **rec), steps=1)
        out[f"{tag}_trace"] = np.array(trace)
        out[f"{tag}_m"] = c.adam.m
        out[f"{tag}_v"] = c.adam.v
    np.savez_compressed(os.path.join(HERE, "train1.npz"), **out)


def golden_f64():
    """The reference's 64-bit shadow mode (init_theta(dtype=float64)): the
    default D = 2 layout (2^12-entry tables) on 500 queries -- encode_batch (f64 X), mlp_forward,
    the relative-L2 loss, mlp_backward with the grid scatter -- and three
    Adam steps on a tiny net (test_training_is_bit_reproducible's recipe)."""
    from nirclab.adam import AdamState, adam_step
    from nirclab.encoding import encode_batch
    from nirclab.losses import loss_relative_l2
    from nirclab.mlp import full_forward, init_theta, make_spec, mlp_backward, mlp_forward

    out = {}
    spec = make_spec(depth=2, table=2 ** 12)
    theta = init_theta(spec, seed=4, dtype=np.float64, out_scale=0.3)
    pos, nrm, alb, rough, dirs = measure_queries(500, seed=11)
    X, ent, wts = encode_batch(spec, theta, pos, nrm, alb, rough, dirs)
    Y, cache = mlp_forward(spec, theta, X, training=True)
    tgt = np.abs(np.random.default_rng(3).normal(size=(500, 3)))
    pdf = np.random.default_rng(4).uniform(0.3, 2.0, 500)
    val, dY = loss_relative_l2(Y, tgt, pdf)
    g = mlp_backward(spec, theta, cache, dY, ent, wts)
    out.update(q=np.concatenate([pos, nrm, alb, rough[:, None], dirs], axis=1), X=X, Y=Y,
               tgt=tgt, pdf=pdf, loss=np.float64(val), g=g, theta0=theta.copy())
    st = AdamState(theta)
    for _ in range(3):
        Y, cache, e2, w2 = full_forward(spec, theta, pos, nrm, alb, rough, dirs, training=True)
        _, dY = loss_relative_l2(Y, tgt, pdf)
        adam_step(st, theta, mlp_backward(spec, theta, cache, dY, e2, w2))
    out["theta3"] = theta
    np.savez_compressed(os.path.join(HERE, "f64.npz"), **out)


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


BOX = """
camera { position 0.5 0.5 -1.4  look_at 0.5 0.5 0.5  up 0 1 0
         fov 39  resolution 16 16 }
material w { kind lambert  albedo 0.7 0.7 0.7 }
material l { kind lambert  albedo 0 0 0  emit 10 10 10 }
quad floor   { material w  p0 0 0 0  p1 1 0 0  p2 1 0 1  p3 0 0 1 }
quad ceiling { material w  p0 0 1 0  p1 0 1 1  p2 1 1 1  p3 1 1 0 }
quad back    { material w  p0 0 0 1  p1 1 0 1  p2 1 1 1  p3 0 1 1 }
quad left    { material w  p0 0 0 0  p1 0 0 1  p2 0 1 1  p3 0 1 0 }
quad right   { material w  p0 1 0 0  p1 1 1 0  p2 1 1 1  p3 1 0 1 }
quad lamp    { material l  p0 0.35 0.999 0.35  p1 0.65 0.999 0.35
               p2 0.65 0.999 0.65  p3 0.35 0.999 0.65 }
"""

# a scene with every material and light kind the device path tracer handles
MIXED = """
camera { position 0.5 0.5 -1.6  look_at 0.5 0.45 0.5  up 0 1 0  fov 42  resolution 24 20 }
material w { kind lambert  albedo 0.7 0.7 0.7 }
material r { kind lambert  albedo 0.6 0.1 0.1 }
material m { kind mirror  albedo 0.9 0.9 0.9 }
material g { kind conductor  albedo 0.9 0.6 0.3  roughness 0.3 }
material l { kind lambert  albedo 0 0 0  emit 8 7 6 }
quad floor   { material w  p0 0 0 0  p1 1 0 0  p2 1 0 1  p3 0 0 1 }
quad back    { material g  p0 0 0 1  p1 1 0 1  p2 1 1 1  p3 0 1 1 }
quad left    { material r  p0 0 0 0  p1 0 0 1  p2 0 1 1  p3 0 1 0 }
quad right   { material m  p0 1 0 0  p1 1 1 0  p2 1 1 1  p3 1 0 1 }
sphere ball  { material w  center 0.35 0.2 0.5  radius 0.2 }
sphere bulb  { material l  center 0.7 0.85 0.45  radius 0.08 }
environment { kind sky  zenith 0.3 0.4 0.8  horizon 0.9 0.9 0.9  ground 0.2 0.2 0.2 }
"""


def golden_scenes():
    """sha1 of every pack array of the builtin scenes and the test scenes."""
    import hashlib
    import json

    from nirclab.scene import load_builtin, load_scene

    out = {}
    scenes = {n: load_builtin(n) for n in ("cornell", "furnace", "occlusion", "teleport")}
    scenes["teleport@50"] = load_builtin("teleport").at_frame(50)
    scenes["BOX"] = load_scene(BOX)
    scenes["MIXED"] = load_scene(MIXED)
    for name, sc in scenes.items():
        d = {}
        for f in sc.pack._fields:
            a = np.ascontiguousarray(np.asarray(getattr(sc.pack, f)))
            d[f] = [str(a.dtype), list(a.shape), hashlib.sha1(a.tobytes()).hexdigest()]
        d["camera"] = hashlib.sha1(np.asarray(sc.camera).tobytes()).hexdigest()
        out[name] = d
    with open(os.path.join(HERE, "scene_packs.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def golden_render():
    """PT and two-level renders (images + path lengths) from the reference."""
    from nirclab.caches import Cache
    from nirclab.estimators import EstimatorConfig, render, render_two_level
    from nirclab.scene import load_builtin, load_scene

    out = {}
    box = load_scene(BOX)
    mixed = load_scene(MIXED)
    corn = load_builtin("cornell")
    jobs = [("box_pt", box, EstimatorConfig(mode="pt"), None, 5, 2),
            ("mixed_pt", mixed, EstimatorConfig(mode="pt"), None, 3, 2),
            ("corn_pt", corn, EstimatorConfig(mode="pt"), None, 0, 1)]
    cbox = Cache.create("nirc", box, seed=9, init="random")
    cmix = Cache.create("nirc", mixed, seed=2, init="random")
    ccor = Cache.create("nirc", corn, seed=1, init="random")
    jobs += [("box_tl", box, EstimatorConfig(mode="two-level", nc=(8, 4, 4)), cbox, 5, 2),
             ("mixed_tl", mixed, EstimatorConfig(mode="two-level", nc=(6, 3, 2)), cmix, 3, 2),
             ("corn_tl", corn, EstimatorConfig(mode="two-level", nc=(8,), max_cache_vertices=1),
              ccor, 0, 1)]
    for tag, sc, cfg, cache, seed, spp in jobs:
        r = render(sc, cfg, cache=cache, seed=seed, spp=spp)
        out[f"{tag}_image"] = r.image
        out[f"{tag}_var"] = r.sample_var
        out[f"{tag}_plen"] = r.path_length
    # zero cache: bit-identical to PT (tests/test_estimators.py:157-166)
    zc = Cache.create("nirc", box, seed=3)
    out["box_tl_zero_forced"] = render_two_level(box, zc, seed=5, spp=2, force_cache=True).image
    np.savez_compressed(os.path.join(HERE, "render.npz"), **out)


def golden_collect():
    """Training records (caches.py:87-131) on the BOX, MIXED and Cornell scenes."""
    from nirclab.caches import collect_training_records
    from nirclab.scene import load_builtin, load_scene

    out = {}
    for tag, sc, count, seed, frame, kind in (
            ("box", load_scene(BOX), 40, 5, 3, "nirc"),
            ("boxfull", load_scene(BOX), 40, 5, 3, "nirc_full"),
            ("mixed", load_scene(MIXED), 60, 2, 1, "nirc"),
            ("corn", load_builtin("cornell"), 103, 0, 0, "nirc"),
            ("boxnrc", load_scene(BOX), 40, 5, 3, "nrc"),
            ("mixednrc", load_scene(MIXED), 60, 2, 1, "nrc"),
            ("mixednvc", load_scene(MIXED), 60, 2, 1, "nvc"),
            ("mixedenv", load_scene(MIXED), 60, 7, 2, "nirc_env")):
        rec = collect_training_records(sc, seed, count, kind=kind, frame=frame)
        for k in ("pos", "ns", "alb", "rough", "dirs", "target", "pdf"):
            out[f"{tag}_{k}"] = getattr(rec, k)
    np.savez_compressed(os.path.join(HERE, "collect.npz"), **out)


def teleport_text(res=128):
    """The builtin teleport scene (lamp jumps at frame 40) at res x res."""
    import nirclab

    path = os.path.join(os.path.dirname(nirclab.__file__), "data", "teleport.scene")
    return open(path).read().replace("resolution 48 48", f"resolution {res} {res}")


CONV = dict(frames=64, ref_spp=128, res=128)


def golden_convergence():
    """BASELINE config 4 at CPU scale: run_experiment (experiment.py:122-213)
    on teleport at 128^2, two-level with the default nc=(15,5,5), 64 frames of
    online training across the frame-40 light jump; per-frame MRSE against a
    128-spp PT reference, rVar, path length and training loss."""
    import tempfile

    from nirclab.config import RunConfig
    from nirclab.experiment import run_experiment
    from nirclab.scene import load_scene

    sc = load_scene(teleport_text(CONV["res"]))
    with tempfile.TemporaryDirectory() as d:
        cfg = RunConfig(scene="teleport", mode="two-level", frames=CONV["frames"], seed=0,
                        out=os.path.join(d, "out"), ref_dir=os.path.join(d, "ref"),
                        ref_spp=CONV["ref_spp"])
        res = run_experiment(cfg, scene=sc)
    rows = res.rows
    np.savez_compressed(os.path.join(HERE, "convergence.npz"),
                        mrse=np.array([r["mrse"] for r in rows]),
                        rvar=np.array([r["rvar"] for r in rows]),
                        plen=np.array([r["avg_path_length"] for r in rows]),
                        loss=np.array([r["train_loss"] for r in rows]),
                        final_image=res.final.image, frames=CONV["frames"],
                        ref_spp=CONV["ref_spp"], res=CONV["res"])


def golden_biased():
    """The biased early-stop family (kernels.py:609-720) through render /
    render_biased: BTH and SPH with a NIRC cache, SPH with an NRC cache, a
    v1 first-vertex map; images, variances and path lengths."""
    from nirclab.caches import Cache
    from nirclab.estimators import EstimatorConfig, render_biased
    from nirclab.scene import load_builtin, load_scene

    out = {}
    box = load_scene(BOX)
    mixed = load_scene(MIXED)
    corn = load_builtin("cornell")
    jobs = []
    for tag, sc, seed in (("box", box, 4), ("mixed", mixed, 6), ("corn", corn, 1)):
        w, h = int(sc.camera[14]), int(sc.camera[15])
        v1 = (np.arange(w * h) % 3 == 0).astype(np.uint8)
        nirc = Cache.create("nirc", sc, seed=seed, init="random")
        nrc = Cache.create("nrc", sc, seed=seed + 1, init="random")
        jobs += [(f"{tag}_bth", sc, EstimatorConfig(mode="biased-nirc-bth", nbias=5), nirc, None),
                 (f"{tag}_nsph", sc, EstimatorConfig(mode="biased-nirc-sph", nbias=7), nirc, v1),
                 (f"{tag}_rsph", sc, EstimatorConfig(mode="biased-nrc-sph"), nrc, v1)]
    for tag, sc, cfg, cache, v1 in jobs:
        r = render_biased(sc, cache, cfg, seed=3, spp=2, frame=1, v1_map=v1)
        out[f"{tag}_image"] = r.image
        out[f"{tag}_var"] = r.sample_var
        out[f"{tag}_plen"] = r.path_length
    np.savez_compressed(os.path.join(HERE, "biased.npz"), **out)


def golden_snapshot():
    """NNCACHE1 files written by the reference's Cache.save
    (caches.py:256-295, snapshot.py:31-49) for a small cache on the BOX:
    fresh, and after one collect + train_frame (m, v, t, frame non-trivial)."""
    from nirclab.caches import Cache
    from nirclab.scene import load_scene

    box = load_scene(BOX)
    c = Cache.create("nirc", box, seed=11, table_log2=10, depth=2)
    c.save(os.path.join(HERE, "snapshot_fresh.nncache"))
    rec = c.collect(count=40, frame=0)
    c.train_frame(rec, steps=2)
    c.save(os.path.join(HERE, "snapshot_trained.nncache"))


def golden_api():
    """Per-interaction API of the reference on the BOX: estimate_Lc /
    estimate_Lr (estimators.py:281-320), sample_incident_targets
    (caches.py:134-155), pt_radiance (estimators.py:240-257), encode +
    mlp_forward_s (encoding.py:170-192, mlp.py:160-192)."""
    from nirclab.caches import Cache, sample_incident_targets
    from nirclab.encoding import encode
    from nirclab.estimators import estimate_Lc, estimate_Lr, pt_radiance
    from nirclab.mlp import mlp_forward_s
    from nirclab.scene import load_scene

    box = load_scene(BOX)
    cache = Cache.create("nirc", box, seed=9, init="random")
    it = box.intersect(np.array([0.5, 0.5, 0.5]), np.array([0.0, -1.0, 0.0]))
    out = {"Lc": estimate_Lc(box, it, cache, n_c=8, seed=3, stream=1),
           "Lr": estimate_Lr(box, it, cache, n_r=3, seed=2, stream=0)}
    d = np.array([0.3, -0.4, 0.5])
    d /= np.linalg.norm(d)
    out["sit"], out["sit_full"] = sample_incident_targets(
        box, [0.5, 0.5, 0.5], d, seed=5, count=6, prev_pdf=0.3, prev_ns=(0.0, 1.0, 0.0),
        frame=2)
    # the reference test's pixels (tests/test_estimators.py:147-152).  Its
    # pt_radiance builds the key in interpreted Python: keys >= 2^63 overflow
    # the jitted rand_uniform, and for frame != 0 it disagrees with its own
    # render_kernel (which ours matches: the convergence run pins the walks)
    pix = [(0, 0, 0), (7, 3, 0), (15, 15, 0)]
    out["pix"] = np.array(pix)
    out["ptr"] = np.array([pt_radiance(box, ix, iy, seed=11, sample=s, frame=0)
                           for ix, iy, s in pix])
    surf = (np.array([0.3, 0.2, 0.7]), np.array([0.0, 1.0, 0.0]), np.array([0.7, 0.7, 0.7]), 1.0)
    x = encode(surf, d, cache)
    out["x"] = x
    mw = int(max(cache.spec.dims))
    out["y"] = np.array(mlp_forward_s(cache.spec, cache.theta, x.astype(np.float32),
                                      np.zeros(mw, np.float32), np.zeros(mw, np.float32)))
    # estimate_env_direct (estimators.py:323-348) on MIXED's sky, NIRC and
    # NVC caches
    from nirclab.estimators import estimate_env_direct

    mixed = load_scene(MIXED)
    itm = mixed.intersect(np.array([0.6, 0.5, 0.3]), np.array([0.0, -1.0, 0.0]))
    for kind in ("nirc", "nvc"):
        cm = Cache.create(kind, mixed, seed=6, init="random")
        out[f"env_{kind}"] = estimate_env_direct(mixed, cm, itm, n_c=8, n_r=5, seed=4,
                                                 stream=2)
    np.savez_compressed(os.path.join(HERE, "api.npz"), **out)


def golden_baseline():
    """The control-variate baselines' integrand sampler (baselines.py:426-431
    over kernels.py:342-421) and the cache evaluation at its live draws
    (_nirc_grid_eval, baselines.py:434-446) on the BOX and MIXED scenes."""
    from nirclab.baselines import _integrand_round, _nirc_grid_eval
    from nirclab.caches import Cache
    from nirclab.caches import _path_arrays
    from nirclab.scene import load_scene

    out = {}
    for tag, sc, seed, frame, k_ in (("box", load_scene(BOX), 3, 0, 4),
                                     ("box2", load_scene(BOX), 3, 2, 4),
                                     ("mixed", load_scene(MIXED), 1, 5, 6)):
        w, h = int(sc.camera[14]), int(sc.camera[15])
        p_ = w * h
        o = dict(dir=np.zeros((p_, k_, 3)), f=np.zeros((p_, k_, 3)),
                 frc=np.zeros((p_, k_, 3)), pdf=np.zeros((p_, k_)),
                 valid=np.zeros(p_, np.uint8), spos=np.zeros((p_, 3)),
                 sns=np.zeros((p_, 3)), salb=np.zeros((p_, 3)), srough=np.zeros(p_))
        scratch = [a[0] for a in _path_arrays(1).values()]
        _integrand_round(sc, seed, frame, k_, scratch, o)
        for k, v in o.items():
            out[f"{tag}_{k}"] = v
        cache = Cache.create("nirc", sc, seed=4, init="random")
        out[f"{tag}_grid"] = _nirc_grid_eval(cache, o, o["pdf"] > 0.0)
    np.savez_compressed(os.path.join(HERE, "baseline.npz"), **out)


def golden_big():
    """A scene past HOST_BVH_MAX (tests/big_scene.py): the reference's
    build_bvh arrays and its PT / two-level renders."""
    sys.path.insert(0, os.path.dirname(HERE))
    from big_scene import big_scene_text
    from nirclab.caches import Cache
    from nirclab.estimators import EstimatorConfig, render
    from nirclab.scene import load_scene

    sc = load_scene(big_scene_text())
    p = sc.pack
    out = {k: np.asarray(getattr(p, k)) for k in ("bvh_lo", "bvh_hi", "bvh_a", "bvh_b",
                                                   "bvh_prim")}
    r = render(sc, EstimatorConfig(mode="pt"), seed=5, spp=2)
    out["pt_image"], out["pt_plen"] = r.image, r.path_length
    cache = Cache.create("nirc", sc, seed=9, init="random")
    r = render(sc, EstimatorConfig(mode="two-level", nc=(8, 4), max_cache_vertices=2), cache=cache,
               seed=5, spp=2)
    out["tl_image"], out["tl_plen"] = r.image, r.path_length
    np.savez_compressed(os.path.join(HERE, "big.npz"), **out)


def _corn_text(res, emit_scale=1.0):
    """The reference's Cornell box edited like tests/scene_texts.py."""
    import nirclab

    sys.path.insert(0, os.path.dirname(HERE))
    from scene_texts import edit_scene

    path = os.path.join(os.path.dirname(nirclab.__file__), "data", "cornell.scene")
    return edit_scene(open(path).read(), res, emit_scale)


def golden_trained():
    """Caches TRAINED by the reference ("a trained
    Cornell snapshot"): collect + train_frame(steps=4) per frame on the
    Cornell box at 64^2 (D = 2, the cfg2 network, 24 frames) and on a
    Cornell box with a 100x brighter lamp (D = 4, 16 frames).  Stores the
    trained theta, the reference's full_forward on 4096 queries inside each
    cache's bounding box, a range-stress variant of the D = 2 net (first
    layer x 2^17, output layer x 2^-17: hidden activations far beyond the
    fp16 range) with its reference outputs, and two-level renders with the
    trained caches."""
    from nirclab.caches import Cache
    from nirclab.estimators import EstimatorConfig, render
    from nirclab.mlp import full_forward, mlp_forward
    from nirclab.encoding import encode_batch
    from nirclab.scene import load_scene

    out = {}
    n = 4096
    for tag, scale, depth, frames in (("corn", 1.0, 2, 24), ("bright", 100.0, 4, 16)):
        sc = load_scene(_corn_text(64, scale))
        c = Cache.create("nirc", sc, seed=5, depth=depth)
        for f in range(frames):
            rec = c.collect(frame=f)
            c.train_frame(rec, steps=4)
        spec = c.spec
        pos, nrm, alb, rough, dirs = measure_queries(n, seed=7)
        bb_min = np.asarray(spec.bb_min, float)
        bb_ext = 1.0 / np.asarray(spec.bb_inv, float)
        pos = bb_min + pos * bb_ext
        out[f"{tag}_theta"] = c.theta.copy()
        out[f"{tag}_bb_min"] = bb_min
        out[f"{tag}_bb_ext"] = bb_ext
        out[f"{tag}_q"] = np.concatenate([pos, nrm, alb, rough[:, None], dirs], axis=1)
        out[f"{tag}_Y"] = full_forward(spec, c.theta, pos, nrm, alb, rough, dirs)
        out[f"{tag}_frame"] = np.int64(c.frame)
        r = render(sc, EstimatorConfig(mode="two-level", nc=(8,), max_cache_vertices=1), cache=c,
                   seed=3, spp=1, frame=c.frame)
        out[f"{tag}_tl_image"] = r.image
        out[f"{tag}_tl_plen"] = r.path_length
        if tag == "corn":
            th = c.theta.copy()
            w0, b0 = int(spec.w_off[0]), int(spec.b_off[0])
            th[w0: b0 + int(spec.dims[1])] *= np.float32(2.0 ** 17)
            wl = int(spec.w_off[-1])
            th[wl:] *= np.float32(2.0 ** -17)
            X, _, _ = encode_batch(spec, th, pos, nrm, alb, rough, dirs)
            out["stress_theta_scale"] = np.float64(2.0 ** 17)
            out["stress_Y"] = mlp_forward(spec, th, X)
            h1 = np.maximum(X @ th[w0: w0 + int(spec.dims[0]) * int(spec.dims[1])].reshape(
                int(spec.dims[1]), int(spec.dims[0])).T + th[b0: b0 + int(spec.dims[1])], 0.0)
            out["stress_h1_max"] = np.float64(h1.max())
    np.savez_compressed(os.path.join(HERE, "trained.npz"), **out)


if __name__ == "__main__" and len(sys.argv) > 1:
    if "trained" in sys.argv:
        golden_trained()
    if "train1" in sys.argv:
        golden_train1()
    if "f64" in sys.argv:
        golden_f64()
    if "big" in sys.argv:
        golden_big()
    if "baseline" in sys.argv:
        golden_baseline()
    if "api" in sys.argv:
        golden_api()
    if "snapshot" in sys.argv:
        golden_snapshot()
    if "biased" in sys.argv:
        golden_biased()
    if "convergence" in sys.argv:
        golden_convergence()
    if "scenes" in sys.argv:
        golden_scenes()
    if "render" in sys.argv:
        golden_render()
    if "collect" in sys.argv:
        golden_collect()
