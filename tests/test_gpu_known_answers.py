"""Known-answer tests of the device walks and record collection, after the
reference's own record / incident-target tests (tests/test_caches.py:100-185
of the reference), on scenes of our own with analytic answers:

* a walk aimed straight at a lamp gives the deterministic MIS-weighted
  emission (balance heuristic against the known next-event pdf) and the raw
  emission in the "full" variant;
* one bounce off a Lambert wall under a rectangular lamp: the mean incident
  radiance is rho/pi * L_e * (the lamp's cosine-weighted solid angle, the
  parallel-rectangle form factor);
* records in a black scene carry zero targets; Lambert records carry
  pdf = cos / pi; full-emission targets dominate MIS targets; directions
  and normals are unit and on the shading side;
* NVC / env records need an environment (ConfigError), visibility targets
  are 0 / 1 and the env-radiance kind is visibility times the sky;
* an unknown record kind is a ConfigError.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

# a 0.6 x 0.6 lamp at height 0.8, facing down (normal -y), emitting (6, 2, 1)
LAMP = """
camera { position 0.5 -2 0.5  look_at 0.5 0 0.5  up 0 0 1  fov 35  resolution 6 6 }
material em { kind lambert  albedo 0 0 0  emit 6 2 1 }
quad lamp { material em  p0 0.2 0.8 0.2  p1 0.8 0.8 0.2  p2 0.8 0.8 0.8  p3 0.2 0.8 0.8 }
"""

# the same lamp above a Lambert floor of albedo 0.45
FLOOR_LAMP = """
camera { position 0.5 0.5 -1.5  look_at 0.5 0.2 0.5  up 0 1 0  fov 40  resolution 6 6 }
material fl { kind lambert  albedo 0.45 0.45 0.45 }
material em { kind lambert  albedo 0 0 0  emit 3 3 3 }
quad floor { material fl  p0 0 0 0  p1 1 0 0  p2 1 0 1  p3 0 0 1 }
quad lamp { material em  p0 0.2 0.8 0.2  p1 0.8 0.8 0.2  p2 0.8 0.8 0.8  p3 0.2 0.8 0.8 }
"""

ROOM = """
camera { position 0.5 0.5 -1.4  look_at 0.5 0.5 0.5  up 0 1 0  fov 39  resolution 8 8 }
material w { kind lambert  albedo 0.6 0.5 0.4 }
material l { kind lambert  albedo 0 0 0  emit EMIT }
quad floor   { material w  p0 0 0 0  p1 1 0 0  p2 1 0 1  p3 0 0 1 }
quad ceiling { material w  p0 0 1 0  p1 0 1 1  p2 1 1 1  p3 1 1 0 }
quad back    { material w  p0 0 0 1  p1 1 0 1  p2 1 1 1  p3 0 1 1 }
quad left    { material w  p0 0 0 0  p1 0 0 1  p2 0 1 1  p3 0 1 0 }
quad right   { material w  p0 1 0 0  p1 1 1 0  p2 1 1 1  p3 1 0 1 }
quad lamp    { material l  p0 0.3 0.999 0.3  p1 0.7 0.999 0.3
               p2 0.7 0.999 0.7  p3 0.3 0.999 0.7 }
"""


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _scene(text):
    from paper_2412_04634_b200.scene import load_scene

    return load_scene(text)


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _form_factor_corner(a, b, h):
    """Integral of cos_r cos_l / d^2 over an a x b rectangle in a plane at
    height h parallel to the receiver, one rectangle corner straight above
    the receiver (the classic differential-area-to-rectangle form factor
    times pi)."""
    ra, rb = np.hypot(a, h), np.hypot(b, h)
    return 0.5 * (a / ra * np.arctan(b / ra) + b / rb * np.arctan(a / rb))


def test_walk_straight_at_lamp_is_exact(cuda):
    from paper_2412_04634_b200.caches import sample_incident_targets

    sc = _scene(LAMP)
    prev_pdf = 0.35
    # two lamp triangles of area 0.18 each, picked with probability 1/2;
    # at distance 0.8 head-on the solid-angle pdf is (1/2)(1/0.18) d^2 / cos
    p_nee = 0.5 / 0.18 * 0.8 * 0.8 / 1.0
    w = prev_pdf / (prev_pdf + p_nee)
    out, full = sample_incident_targets(sc, (0.4, 0.0, 0.55), (0.0, 1.0, 0.0), seed=3,
                                        count=48, prev_pdf=prev_pdf, prev_ns=(0.0, 1.0, 0.0))
    assert np.max(np.abs(out - w * np.array([6.0, 2.0, 1.0]))) < 1e-9
    assert np.max(np.abs(full - np.array([6.0, 2.0, 1.0]))) < 1e-12


def test_one_bounce_mean_matches_form_factor(cuda):
    from paper_2412_04634_b200.caches import sample_incident_targets

    sc = _scene(FLOOR_LAMP)
    n = 200_000
    out, _ = sample_incident_targets(sc, (0.5, 0.3, 0.5), (0.0, -1.0, 0.0), seed=9, count=n)
    # the floor point (0.5, 0, 0.5) sits under the lamp centre: four
    # 0.3 x 0.3 quadrants at height 0.8
    expect = 0.45 / np.pi * 3.0 * 4.0 * _form_factor_corner(0.3, 0.3, 0.8)
    mean = out.mean(axis=0)
    se = out.std(axis=0) / np.sqrt(n)
    assert np.all(np.abs(mean - expect) < max(5 * se.max(), 0.005 * expect)), (mean, expect)


def test_record_known_answers(cuda):
    from paper_2412_04634_b200.records import collect_training_records

    lit = _scene(ROOM.replace("EMIT", "8 8 8"))
    dark = _scene(ROOM.replace("EMIT", "0 0 0"))
    for kind in ("nirc", "nrc", "nirc_full"):
        rec = collect_training_records(lit, seed=1, count=70, kind=kind)
        n = len(rec)
        assert n > 70
        tgt = _np(rec.target)
        dirs = _np(rec.dirs)
        ns = _np(rec.ns)
        pdf = _np(rec.pdf)
        assert tgt.shape == (n, 3) and np.all(np.isfinite(tgt)) and np.all(tgt >= 0)
        assert np.allclose(np.linalg.norm(dirs, axis=1), 1.0, atol=1e-9)
        assert np.allclose(np.linalg.norm(ns, axis=1), 1.0, atol=1e-9)
        cos = np.einsum("ij,ij->i", dirs, ns)
        assert np.all(cos > 0)
        if kind != "nrc":  # every surface is Lambert: the recorded pdf is cos / pi
            assert np.max(np.abs(pdf - cos / np.pi)) < 1e-12
        else:  # NRC records: (wo, the sampling pdf of the path's arrival)
            assert np.all(pdf > 0)
        blk = collect_training_records(dark, seed=1, count=70, kind=kind)
        bt = _np(blk.target)
        assert len(blk) > 0 and np.all(bt == 0.0)
    a = collect_training_records(lit, seed=4, count=60, kind="nirc")
    b = collect_training_records(lit, seed=4, count=60, kind="nirc_full")
    ta = _np(a.target)
    tb = _np(b.target)
    assert len(a) == len(b)
    assert np.all(tb >= ta - 1e-12) and np.any(tb > ta + 1e-9)


def test_env_record_kinds(cuda):
    from paper_2412_04634_b200.errors import ConfigError
    from paper_2412_04634_b200.records import collect_training_records
    from paper_2412_04634_b200.scene import load_builtin

    room = _scene(ROOM.replace("EMIT", "8 8 8"))
    for kind in ("nvc", "nirc_env"):
        with pytest.raises(ConfigError):
            collect_training_records(room, seed=1, count=10, kind=kind)
    with pytest.raises(ConfigError):
        collect_training_records(room, seed=1, count=10, kind="photon")
    sc = load_builtin("occlusion")
    vis = collect_training_records(sc, seed=2, count=80, kind="nvc")
    rad = collect_training_records(sc, seed=2, count=80, kind="nirc_env")
    v = _np(vis.target)
    r = _np(rad.target)
    assert len(vis) == len(rad) > 0
    assert set(np.unique(v)) <= {0.0, 1.0}
    assert np.array_equal(v[:, 0], v[:, 1]) and np.array_equal(v[:, 1], v[:, 2])
    lit = v[:, 0] == 1.0
    assert np.all(r[~lit] == 0.0) and np.all(r[lit] > 0.0)


def test_divergence_and_nonfinite_guards(cuda, tmp_path):
    """The reference's guards (caches.py:347-353, mlp.py:104-105,
    adam.py:22-24; its tests test_caches.py:304-312, test_neural.py:178-183):
    a non-finite loss raises DivergenceError after dumping the cache state
    (one .nncache, its path in the message) and leaves the frame counter;
    mlp_forward refuses a non-finite theta."""
    from paper_2412_04634_b200.caches import Cache, Records
    from paper_2412_04634_b200.errors import DivergenceError
    from paper_2412_04634_b200.mlp import init_theta, make_spec, mlp_forward

    sc = _scene(ROOM.replace("EMIT", "8 8 8"))
    cache = Cache.create("nirc", sc, seed=7, loss="l2")
    cache.snapshot_dir = str(tmp_path)
    rng = np.random.default_rng(3)
    n = 64
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    rec = Records(kind="nirc", frame=0, pos=rng.uniform(size=(n, 3)), ns=nrm,
                  alb=rng.uniform(size=(n, 3)), rough=np.ones(n), dirs=nrm.copy(),
                  target=np.full((n, 3), np.inf), pdf=np.full(n, 0.3))
    frame0 = cache.frame
    with pytest.raises(DivergenceError) as err:
        cache.train_frame(rec)
    dumps = list(tmp_path.iterdir())
    assert len(dumps) == 1 and str(dumps[0]) in str(err.value)
    assert err.value.snapshot_path == str(dumps[0])
    assert cache.frame == frame0
    spec = make_spec(depth=2)
    theta = init_theta(spec, seed=1)
    theta[spec.grid_len + 3] = np.nan
    with pytest.raises(DivergenceError):
        mlp_forward(spec, theta, np.zeros((1, spec.in_dim), np.float32))


def _const_records(n, seed, target, pdf=1.0):
    from paper_2412_04634_b200.caches import Records

    rng = np.random.default_rng(seed)
    ns = rng.normal(size=(n, 3))
    ns /= np.linalg.norm(ns, axis=1, keepdims=True)
    dirs = rng.normal(size=(n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return Records(kind="nirc", frame=0, pos=rng.uniform(0, 1, (n, 3)), ns=ns,
                   alb=np.full((n, 3), 0.45), rough=np.ones(n), dirs=dirs,
                   target=np.broadcast_to(np.asarray(target, float), (n, 3)).copy(),
                   pdf=np.full(n, pdf))


def test_training_learns_constant_and_zero_targets(cuda):
    """Online training behaves like the reference's (its
    tests/test_caches.py:277-301): constant targets are learned to within 1 %
    of their mean after 2000 optimizer steps from the zero-initialised output
    layer, and zero targets drive a random cache's output down."""
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.mlp import full_forward

    sc = _scene(ROOM.replace("EMIT", "8 8 8"))
    target = np.array([0.6, 0.45, 0.25])
    cache = Cache.create("nirc", sc, seed=6)
    rec = _const_records(256, 8, target)
    for _ in range(500):  # 2000 optimizer steps
        cache.train_frame(rec)
    pred = np.asarray(full_forward(cache.spec, cache.theta, rec.pos, rec.ns, rec.alb, rec.rough,
                                   rec.dirs))
    assert np.all(np.abs(pred.mean(axis=0) - target) / target < 0.01)

    cache = Cache.create("nirc", sc, seed=5, init="random", loss="l2")
    rec = _const_records(512, 21, 0.0)
    before = np.asarray(full_forward(cache.spec, cache.theta, rec.pos, rec.ns, rec.alb,
                                     rec.rough, rec.dirs))
    for _ in range(100):
        cache.train_frame(rec)
    after = np.asarray(full_forward(cache.spec, cache.theta, rec.pos, rec.ns, rec.alb, rec.rough,
                                    rec.dirs))
    assert np.abs(before).mean() > 1e-3
    assert np.abs(after).mean() < 1e-3


def test_path_tracer_analytic_scenes(cuda):
    """Analytic answers of the device path tracer (the reference's
    tests/test_estimators.py:124-144 on scenes of our own): an empty scene
    is exactly its constant environment with zero path length; a huge
    Lambert floor under a unit sky reflects its albedo; the builtin furnace
    (unit albedo in a unit sky) converges to 1 everywhere."""
    from paper_2412_04634_b200.estimators import EstimatorConfig, render
    from paper_2412_04634_b200.scene import load_builtin

    empty = _scene("""
camera { position 0 0 0  look_at 0 1 1  up 0 1 0  fov 50  resolution 10 6 }
environment { kind constant  color 1.7 1.7 1.7 }
""")
    out = render(empty, EstimatorConfig(mode="pt"), seed=4, spp=3)
    assert np.all(out.image == 1.7)
    assert out.avg_path_length == 0.0
    floor = _scene("""
camera { position 0 30 0.001  look_at 0 0 0  up 0 1 0  fov 25  resolution 10 10 }
material m { kind lambert  albedo 0.35 0.35 0.35 }
quad ground { material m  p0 -400 0 -400  p1 400 0 -400  p2 400 0 400  p3 -400 0 400 }
environment { kind constant  color 1.0 1.0 1.0 }
""")
    out = render(floor, EstimatorConfig(mode="pt"), seed=2, spp=64)
    assert np.max(np.abs(out.image - 0.35)) < 5e-3
    out = render(load_builtin("furnace"), EstimatorConfig(mode="pt"), seed=1, spp=256)
    assert abs(float(out.image.mean()) - 1.0) < 0.01
    assert np.max(np.abs(out.image - 1.0)) < 0.01


def test_nvc_cache_bounds_guard_and_learning(cuda):
    """The visibility cache (NVC, sigmoid head) after the reference's
    tests/test_caches.py:236-250,343-353: outputs in (0, 1), queries need an
    environment light, and online training on the occlusion scene learns
    ray-cast visibility of fresh (surface, direction) pairs."""
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.errors import ConfigError
    from paper_2412_04634_b200.mlp import full_forward
    from paper_2412_04634_b200.records import collect_training_records
    from paper_2412_04634_b200.scene import load_builtin

    sky = load_builtin("occlusion")
    cache = Cache.create("nvc", sky, seed=2, init="random")
    it = sky.intersect([0.0, 3.0, 0.0], [0.0, -1.0, 0.0])
    rng = np.random.default_rng(4)
    dirs = rng.normal(size=(50, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    out = cache.nvc_query(it, dirs)
    assert np.all(out > 0.0) and np.all(out < 1.0)
    room = _scene(ROOM.replace("EMIT", "8 8 8"))
    no_env = Cache.create("nvc", room, seed=2)
    with pytest.raises(ConfigError):
        no_env.nvc_query(room.intersect([0.5, 0.5, 0.5], [0.0, -1.0, 0.0]), dirs)

    cache = Cache.create("nvc", sky, seed=13)
    for f in range(256):
        rec = cache.collect()
        if len(rec):
            cache.train_frame(rec)
    rec = collect_training_records(sky, seed=999, count=200, kind="nvc")
    pred = full_forward(cache.spec, cache.theta, rec.pos, rec.ns, rec.alb, rec.rough, rec.dirs)
    mae = float((pred[:, 0].double() - rec.target[:, 0]).abs().mean())
    assert mae < 0.12
