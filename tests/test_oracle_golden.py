"""The CPU oracle against the reference's own outputs (tests/golden/*.npz).

This pins the oracle: every later GPU parity test trusts it only because
these checks hold bit for bit (integer/bit-exact work) or within the
reference's own float tolerances.
"""

import numpy as np
import pytest

import nirc_oracle as O


def test_rng_known_answers():
    # splitmix64 chain, rng.py:59-73 (values printed by the reference)
    assert O.mix64_int(5) == 7134611160154358618
    assert O.stream_key(0, O.P_SHUFFLE, 0, 3, 0) == 2681611406235024285


def test_measure_queries_match_reference(golden):
    g = golden("encode_forward")
    pos, nrm, alb, rough, dirs = O.measure_queries(4096)
    for a, k in ((pos, "pos"), (nrm, "nrm"), (alb, "alb"), (rough, "rough"), (dirs, "dirs")):
        assert np.array_equal(a, g[k]), k


def test_encode_bit_exact_against_reference(golden):
    g = golden("encode_forward")
    spec = O.Spec(depth=2)
    theta = O.init_theta(spec, seed=1, out_scale=0.1)
    X, ent, wts = O.encode_batch(spec, theta, g["pos"], g["nrm"], g["alb"], g["rough"],
                                 g["dirs"])
    assert np.array_equal(ent, g["entries"].astype(np.int64))
    assert np.array_equal(wts, g["weights"])
    assert np.array_equal(X, g["X"])


@pytest.mark.parametrize("depth", [2, 4])
def test_forward_matches_reference(golden, depth):
    g = golden("encode_forward")
    spec = O.Spec(depth=depth)
    theta = O.init_theta(spec, seed=1, out_scale=0.1)
    Y = O.mlp_forward(spec, theta, g["X"])
    np.testing.assert_allclose(Y, g[f"Y_d{depth}"], rtol=1e-5, atol=1e-7)


def test_grid_vertex_identity_known_answer():
    # tests/test_neural.py:52-64 of the reference
    spec = O.Spec(levels=1, table=64, base_res=4, max_res=4, bands=1, depth=1, width=4)
    theta = O.init_theta(spec, seed=1).astype(np.float32)
    theta[: spec.grid_len] = np.random.default_rng(1).random(spec.grid_len)
    X, _, _ = O.encode_batch(spec, theta, np.array([[0.25, 0.5, 0.75]]),
                             np.array([[0.0, 0, 1]]), np.full((1, 3), 0.5), np.ones(1),
                             np.array([[0.0, 0, 1]]))
    h = (1 * 1 ^ 2 * 2654435761 ^ 3 * 805459861) & 63
    assert X[0, 0] == theta[h * 2] and X[0, 1] == theta[h * 2 + 1]


def test_losses_match_reference(golden):
    g = golden("losses_adam")
    v, gr = O.loss_relative_l2(g["y"], g["t"], g["pdf"])
    assert v == pytest.approx(float(g["rel_val"]), rel=1e-14)
    np.testing.assert_array_equal(gr, g["rel_grad"])
    v, gr = O.loss_l2(g["y"], g["t"], g["pdf"])
    assert v == pytest.approx(float(g["l2_val"]), rel=1e-14)
    np.testing.assert_array_equal(gr, g["l2_grad"])
    # known answers, tests/test_neural.py:259-276
    v, _ = O.loss_relative_l2(np.full((1, 3), 1.0, np.float32), np.full((1, 3), 2.0), np.ones(1))
    assert v == pytest.approx(1.0 / 1.01, rel=1e-6)
    v, _ = O.loss_l2(np.full((1, 3), 1.0), np.full((1, 3), 3.0), np.full(1, 0.5))
    assert v == pytest.approx(8.0)


def test_adam_bit_exact_against_reference(golden):
    g = golden("losses_adam")
    theta = g["theta0"].copy()
    st = O.Adam(theta.size)
    for k, gr in enumerate(g["grads"]):
        st.step(theta, gr)
        assert np.array_equal(theta, g["thetas"][k]), k
    assert st.t == int(g["t_final"]) and st.skipped == int(g["skipped"])


@pytest.mark.parametrize("tag,n", [("small", 3000), ("big", 20000)])
def test_train_steps_match_reference(golden, tag, n):
    g = golden("train_step")
    rec = O.synth_records(n, seed=5)
    assert np.allclose([v.sum() for v in rec.values()], g[f"{tag}_rec_digest"], rtol=0, atol=0)
    spec = O.Spec(table=2 ** 12, depth=4)
    theta = O.init_theta(spec, seed=3)
    adam = O.Adam(spec.theta_len)
    trace = []
    for s in range(2):
        val, idx = O.train_step(spec, theta, adam, rec, seed=7, frame=2, step=s)
        assert np.array_equal(idx, g[f"{tag}_idx{s}"])
        trace.append(val)
    np.testing.assert_allclose(trace, g[f"{tag}_trace"], rtol=1e-6)
    # same math, numpy either side: parameters agree to f32 rounding noise
    np.testing.assert_allclose(theta, g[f"{tag}_theta"], rtol=1e-4, atol=1e-6)
    assert adam.t == int(g[f"{tag}_t"])
