"""Batch consumers of fused inference from the control-variate baselines
 against the reference's own outputs
(tests/golden/baseline.npz from tests/golden/make_golden.py baseline):
integrand_samples_kernel (kernels.py:342-421) through nirc_integrand_samples,
and _nirc_grid_eval (baselines.py:434-446) through the fused full_forward."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

_SRC = open(os.path.join(GOLDEN, "make_golden.py")).read()
SCENES = {"BOX": _SRC.split('BOX = """')[1].split('"""')[0],
          "MIXED": _SRC.split('MIXED = """')[1].split('"""')[0]}
CASES = (("box", "BOX", 3, 0, 4), ("box2", "BOX", 3, 2, 4), ("mixed", "MIXED", 1, 5, 6))
KEYS = ("dir", "f", "frc", "pdf", "valid", "spos", "sns", "salb", "srough")


@pytest.fixture(scope="module")
def scenes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_04634_b200.scene import load_scene

    return {k: load_scene(v) for k, v in SCENES.items()}


def _round(sc, seed, frame, k_):
    from paper_2412_04634_b200.baselines import _integrand_round

    w, h = int(sc.camera[14]), int(sc.camera[15])
    p_ = w * h
    o = dict(dir=np.zeros((p_, k_, 3)), f=np.zeros((p_, k_, 3)), frc=np.zeros((p_, k_, 3)),
             pdf=np.zeros((p_, k_)), valid=np.zeros(p_, np.uint8), spos=np.zeros((p_, 3)),
             sns=np.zeros((p_, 3)), salb=np.zeros((p_, 3)), srough=np.zeros(p_))
    _integrand_round(sc, seed, frame, k_, None, o)
    return o


@pytest.mark.parametrize("tag,scene,seed,frame,k_", CASES)
def test_integrand_round_matches_reference(scenes, golden, tag, scene, seed, frame, k_):
    g = golden("baseline")
    o = _round(scenes[scene], seed, frame, k_)
    np.testing.assert_array_equal(o["valid"], g[f"{tag}_valid"])
    # the same draws are live (pdf > 0) and the walks see the same vertices
    np.testing.assert_array_equal(o["pdf"] > 0, g[f"{tag}_pdf"] > 0)
    for k in ("dir", "frc", "pdf", "spos", "sns", "salb", "srough"):
        np.testing.assert_allclose(o[k], g[f"{tag}_{k}"], rtol=1e-9, atol=1e-12, err_msg=k)
    # integrand samples: f64 walks, FMA-contracted on the device like the
    # reference's fastmath JIT (SURVEY.md 8(c) pixel-estimate calibration)
    np.testing.assert_allclose(o["f"], g[f"{tag}_f"], rtol=1e-8, atol=1e-12)


def test_integrand_round_leaves_untouched_entries(scenes):
    """Missed / mirror pixels and dead draws keep the caller's values, like
    the reference kernel's `continue`s."""
    from paper_2412_04634_b200.baselines import integrand_buffers, integrand_round

    sc = scenes["MIXED"]
    out = integrand_buffers(sc, 3)
    for k in ("dir", "f", "frc"):
        out[k].fill_(7.0)
    integrand_round(sc, 1, 0, 3, out)
    dead = (out["pdf"] <= 0).cpu().numpy()
    assert dead.any()
    for k in ("dir", "f", "frc"):
        assert np.all(out[k].cpu().numpy()[dead] == 7.0)
    # a pixel with no valid primary hit keeps pdf 0 and no surface data
    inval = out["valid"].cpu().numpy() == 0
    assert inval.any() and np.all(out["srough"].cpu().numpy()[inval] == 0.0)


def test_nirc_grid_eval_matches_reference(scenes, golden):
    from paper_2412_04634_b200.baselines import _nirc_grid_eval
    from paper_2412_04634_b200.caches import Cache

    g = golden("baseline")
    for tag, scene, *_ in CASES:
        sc = scenes[scene]
        o = {k: g[f"{tag}_{k}"] for k in KEYS}
        cache = Cache.create("nirc", sc, seed=4, init="random")
        got = _nirc_grid_eval(cache, o, o["pdf"] > 0.0)
        # fused 2xFP16 tcgen05 inference: the fp32 parity bar (rtol 1e-4)
        np.testing.assert_allclose(got, g[f"{tag}_grid"], rtol=1e-4, atol=1e-7, err_msg=tag)
