"""The reference's 64-bit shadow mode on the device:
init_theta(dtype=float64) networks through the same drop-in API --
encode_batch / mlp_forward / losses / mlp_backward + scatter_grid_grad /
adam_step -- against the reference's own f64 outputs (tests/golden/f64.npz),
and the reference's verification recipes run through the shim:
  * the five-point finite-difference gradient check of every parameter
    (gradient_check, mlp.py:227-292; pkg/tests/test_neural.py:223-253,
    relative error < 1e-5);
  * test_training_is_bit_reproducible (pkg/tests/test_neural.py:369-385).
Tolerances: the encoded X bit-exact (same corner-ordered f64 sums, the SH
recurrences in the reference's order); outputs / gradients within 1e-12
relative (BLAS dgemm vs the device's fma order)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_04634_b200 import _lib

    _lib.load()


def tiny_spec(out_act=0, bands=1, depth=2, width=8, levels=2, table=16):
    from paper_2412_04634_b200.mlp import make_spec

    return make_spec(levels=levels, table=table, feats=2, base_res=2, max_res=4, bands=bands,
                     depth=depth, width=width, out_dim=3, out_act=out_act)


def random_batch(seed, n=4):
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3))
    normal = rng.normal(size=(n, 3))
    normal /= np.linalg.norm(normal, axis=1, keepdims=True)
    albedo = rng.random((n, 3))
    rough = rng.random(n)
    dirs = rng.normal(size=(n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    target = rng.random((n, 3))
    pdf = rng.uniform(0.3, 2.0, n)
    return (pos, normal, albedo, rough, dirs), target, pdf


def test_f64_pipeline_matches_reference(nb, golden):
    from paper_2412_04634_b200.encoding import encode_batch
    from paper_2412_04634_b200.losses import loss_relative_l2
    from paper_2412_04634_b200.mlp import make_spec, mlp_backward, mlp_forward

    g = golden("f64")
    spec = make_spec(depth=2, table=2 ** 12)
    th = g["theta0"]
    q = g["q"]
    X, ent, wts = encode_batch(spec, th, q[:, 0:3], q[:, 3:6], q[:, 6:9], q[:, 9].copy(),
                               q[:, 10:13])
    assert X.dtype == np.float64
    assert np.array_equal(X, g["X"])
    Y, cache = mlp_forward(spec, th, X, training=True)
    np.testing.assert_allclose(Y, g["Y"], rtol=1e-12, atol=1e-15)
    val, dY = loss_relative_l2(Y, g["tgt"], g["pdf"])
    assert val == pytest.approx(float(g["loss"]), rel=1e-12)
    grad = mlp_backward(spec, th, cache, dY, ent, wts)
    assert grad.dtype == np.float64
    np.testing.assert_allclose(grad, g["g"], rtol=1e-10, atol=1e-14 * np.abs(g["g"]).max())


def test_f64_adam_steps_match_reference(nb, golden):
    from paper_2412_04634_b200.adam import AdamState, adam_step
    from paper_2412_04634_b200.losses import loss_relative_l2
    from paper_2412_04634_b200.mlp import full_forward, make_spec, mlp_backward

    g = golden("f64")
    spec = make_spec(depth=2, table=2 ** 12)
    th = g["theta0"].copy()
    q = g["q"]
    surf = (q[:, 0:3], q[:, 3:6], q[:, 6:9], q[:, 9].copy(), q[:, 10:13])
    st = AdamState(th)
    for _ in range(3):
        Y, cache, e, w = full_forward(spec, th, *surf, training=True)
        _, dY = loss_relative_l2(Y, g["tgt"], g["pdf"])
        assert adam_step(st, th, mlp_backward(spec, th, cache, dY, e, w))
    np.testing.assert_allclose(th, g["theta3"], rtol=1e-10, atol=1e-13)
    assert st.t == 3


def _kink_free(seed, out_act=0):
    from paper_2412_04634_b200.mlp import full_forward, init_theta

    for attempt in range(20):
        s = seed + 1000 * attempt
        spec = tiny_spec(out_act=out_act)
        theta = init_theta(spec, seed=s, dtype=np.float64, out_scale=0.6)
        surf, target, pdf = random_batch(s + 7)
        _, (_, zs), _, _ = full_forward(spec, theta, *surf, training=True)
        if np.abs(zs.cpu().numpy()).min() > 1e-2:
            return spec, theta, surf, target, pdf
    raise AssertionError("no kink-free configuration found")


@pytest.mark.parametrize("loss_kind", ["l2", "relative_l2", "variance"])
def test_gradients_match_finite_differences(nb, loss_kind):
    """pkg/tests/test_neural.py:240-245 through the device path."""
    from paper_2412_04634_b200.mlp import gradient_check

    for seed in range(10):  # the reference's 10 seeds
        spec, theta, surf, target, pdf = _kink_free(seed)
        err = gradient_check(spec, theta, surf, target, pdf, loss_kind)
        assert err < 1e-5, f"seed {seed}: rel err {err}"


def test_bce_gradient_matches_finite_differences(nb):
    from paper_2412_04634_b200.mlp import gradient_check

    for seed in range(5):  # the reference's 5 seeds
        spec, theta, surf, target, pdf = _kink_free(seed, out_act=1)
        err = gradient_check(spec, theta, surf, target, pdf, "bce")
        assert err < 1e-5, f"seed {seed}: rel err {err}"


def test_training_is_bit_reproducible(nb):
    """pkg/tests/test_neural.py:369-385 verbatim in shape: f64 theta, 3
    full_forward / loss / mlp_backward / adam_step rounds, twice."""
    from paper_2412_04634_b200.adam import AdamState, adam_step
    from paper_2412_04634_b200.losses import loss_relative_l2
    from paper_2412_04634_b200.mlp import full_forward, init_theta, mlp_backward

    def run():
        spec = tiny_spec()
        theta = init_theta(spec, seed=7, dtype=np.float64, out_scale=0.2)
        st = AdamState(theta)
        surf, target, pdf = random_batch(8, n=16)
        for _ in range(3):
            Y, cache, entries, weights = full_forward(spec, theta, *surf, training=True)
            _, dY = loss_relative_l2(Y, target, pdf)
            g = mlp_backward(spec, theta, cache, dY, entries, weights)
            adam_step(st, theta, g)
        return theta

    a = run()
    b = run()
    assert np.array_equal(a, b)


def test_forward_scalar_reference_matches_batch(nb):
    """forward_scalar_reference (mlp.py:195-213) vs the device batch
    forward, f64 and f32 (pkg/tests/test_neural.py:146-158, rtol 1e-6)."""
    from paper_2412_04634_b200.mlp import (forward_scalar_reference, init_theta, make_spec,
                                           mlp_forward)

    spec = make_spec(depth=2, width=16, levels=4, table=64, bands=2)
    for dtype in (np.float64, np.float32):
        theta = init_theta(spec, seed=3, dtype=dtype, out_scale=0.5)
        X = np.random.default_rng(1).random((6, spec.in_dim)).astype(dtype)
        Y = np.asarray(mlp_forward(spec, theta, X))
        for i in range(6):
            np.testing.assert_allclose(Y[i], forward_scalar_reference(spec, theta, X[i]),
                                       rtol=1e-6, atol=1e-7)
