"""Device BVH build: nirc_build_bvh equals the
reference's median-split build_bvh (geometry.py:213-274) node for node --
against the host restatement on builtin, golden and random primitive soups
(ties in the centroid keys, degenerate extents, every leaf-size boundary),
and against the reference's own arrays for the larger scene
(tests/golden/big.npz); that scene then renders (PT and two-level) like the
reference."""

import os

import numpy as np
import pytest
import torch

from big_scene import big_scene_text
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

_SRC = open(os.path.join(GOLDEN, "make_golden.py")).read()
TEXTS = {"BOX": _SRC.split('BOX = """')[1].split('"""')[0],
         "MIXED": _SRC.split('MIXED = """')[1].split('"""')[0]}
KEYS = ("bvh_lo", "bvh_hi", "bvh_a", "bvh_b", "bvh_prim")


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _same(dev, host):
    for k, (x, y) in zip(KEYS, zip(dev, host)):
        assert x.shape == y.shape, k
        np.testing.assert_array_equal(x, y, err_msg=k)


def _soup(nt, ns_, seed, quantise=False):
    rng = np.random.default_rng(seed)
    v0 = rng.uniform(-1, 1, (nt, 3))
    e1 = rng.normal(0, 0.05, (nt, 3))
    e2 = rng.normal(0, 0.05, (nt, 3))
    c = rng.uniform(-1, 1, (ns_, 3))
    r = rng.uniform(0.01, 0.1, ns_)
    if quantise:  # many equal centroid keys: the stable sort's tie order
        v0, c = np.round(v0 * 4) / 4, np.round(c * 4) / 4
        e1, e2 = np.round(e1 * 64) / 64, np.round(e2 * 64) / 64
        r = np.full(ns_, 0.0625)
    return v0, e1, e2, c, r


@pytest.mark.parametrize("n", [0, 1, 4, 5, 6, 7, 8, 9, 16, 17, 33, 100, 1000, 4097])
def test_device_bvh_equals_host_on_soups(cuda, n):
    from paper_2412_04634_b200.scene import build_bvh, build_bvh_device

    for q in (False, True):
        args = _soup(n - n // 4, n // 4, seed=n, quantise=q)
        _same(build_bvh_device(*args), build_bvh(*args))


def test_device_bvh_flat_and_coincident(cuda):
    """Zero extent along axes (argmax's first-on-ties) and coincident
    primitives."""
    from paper_2412_04634_b200.scene import build_bvh, build_bvh_device

    n = 300
    v0 = np.zeros((n, 3))
    v0[:, 0] = np.arange(n) % 7
    e1 = np.tile([0.0, 0.0, 1.0], (n, 1))
    e2 = np.tile([0.0, 1.0, 0.0], (n, 1))
    args = (v0, e1, e2, np.zeros((5, 3)), np.full(5, 0.5))
    _same(build_bvh_device(*args), build_bvh(*args))


def test_device_bvh_on_scenes(cuda):
    from paper_2412_04634_b200.scene import build_bvh_device, load_builtin, load_scene

    scenes = [load_builtin(n) for n in ("cornell", "furnace", "occlusion", "teleport")]
    scenes += [load_scene(t) for t in TEXTS.values()]
    for sc in scenes:
        p = sc.pack
        got = build_bvh_device(p.tri_v0, p.tri_e1, p.tri_e2, p.sph_c, p.sph_r)
        _same(got, [getattr(p, k) for k in KEYS])


def test_big_scene_bvh_and_render_match_reference(cuda, golden):
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.estimators import EstimatorConfig, render
    from paper_2412_04634_b200.scene import HOST_BVH_MAX, load_scene

    g = golden("big")
    sc = load_scene(big_scene_text())
    assert len(sc.pack.tri_v0) + len(sc.pack.sph_c) > HOST_BVH_MAX  # built on the device
    _same([getattr(sc.pack, k) for k in KEYS], [g[k] for k in KEYS])
    r = render(sc, EstimatorConfig(mode="pt"), seed=5, spp=2)
    assert np.array_equal(r.path_length, g["pt_plen"])
    np.testing.assert_allclose(r.image, g["pt_image"], rtol=1e-9, atol=1e-12)
    cache = Cache.create("nirc", sc, seed=9, init="random")
    r = render(sc, EstimatorConfig(mode="two-level", nc=(8, 4), max_cache_vertices=2),
               cache=cache, seed=5, spp=2)
    assert np.array_equal(r.path_length, g["tl_plen"])
    np.testing.assert_allclose(r.image, g["tl_image"], rtol=1e-5, atol=5e-7)
