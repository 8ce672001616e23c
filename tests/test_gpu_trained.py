"""Parity on caches TRAINED by the reference, the 2xFP16 range guard, the
reference's DivergenceError on a non-finite theta, the pinned-host pipeline
and the library's stream-ordered concurrency contract.

Fixtures: tests/golden/trained.npz (make_golden.py ``trained``): a D = 2
Cornell cache trained 24 frames and a D = 4 cache trained 16 frames on a
Cornell box with a 100x lamp, both by nirclab's own collect + train_frame;
the reference's full_forward on 4096 queries inside each bbox; a
range-stress net (first layer x 2^17, output layer x 2^-17: hidden
activations up to 2.2e5, beyond fp16) with the reference's outputs; and
two-level renders with the trained caches.

Tolerances: network outputs rtol 1e-4 (the reference's own scalar-vs-batch
bar, tests/test_neural.py:174) at every precision; two-level images rtol
1e-3 / atol 1e-4 like tests/test_gpu_render.py, path lengths identical.
"""

import numpy as np
import pytest
import torch

import nirc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_04634_b200 import _lib

    _lib.load()


def _spec(g, tag, depth):
    from paper_2412_04634_b200.mlp import make_spec

    return make_spec(depth=depth, bb_min=g[f"{tag}_bb_min"], bb_ext=g[f"{tag}_bb_ext"])


def _rows(q):
    return q[:, 0:3], q[:, 3:6], q[:, 6:9], q[:, 9].copy(), q[:, 10:13]


@pytest.mark.parametrize("precision", [0, 1, 2])
@pytest.mark.parametrize("tag,depth", [("corn", 2), ("bright", 4)])
def test_full_forward_trained_cache(nb, golden, tag, depth, precision):
    """cfg2's forward on a reference-trained cache ("θ =
    init_theta ... and a trained Cornell snapshot")."""
    from paper_2412_04634_b200.mlp import full_forward

    g = golden("trained")
    spec = _spec(g, tag, depth)
    y = full_forward(spec, g[f"{tag}_theta"], *_rows(g[f"{tag}_q"]), precision=precision)
    ref = g[f"{tag}_Y"]
    scale = float(np.abs(ref).max())
    np.testing.assert_allclose(y, ref, rtol=1e-4, atol=1e-6 * scale)


@pytest.mark.parametrize("precision", [0, 2])
def test_full_forward_fp16_range_guard(nb, golden, precision):
    """Hidden activations up to 2.2e5 (beyond fp16's 65504): the 2xFP16
    path flags the affected rows and recomputes them in fp32, so the result
    still matches the reference; 3xTF32 has fp32's range natively."""
    from paper_2412_04634_b200.mlp import full_forward

    g = golden("trained")
    assert float(g["stress_h1_max"]) > 65504.0
    spec = _spec(g, "corn", 2)
    th = g["corn_theta"].copy()
    s = np.float32(float(g["stress_theta_scale"]))
    th[int(spec.w_off[0]): int(spec.b_off[0]) + int(spec.dims[1])] *= s
    th[int(spec.w_off[-1]):] *= np.float32(1.0) / s
    y = full_forward(spec, th, *_rows(g["corn_q"]), precision=precision)
    ref = g["stress_Y"]
    assert np.all(np.isfinite(y))
    np.testing.assert_allclose(y, ref, rtol=1e-4, atol=1e-6 * float(np.abs(ref).max()))


def test_fp16_guard_weights_and_inputs(nb):
    """Weights beyond fp16 (every row recomputed) and a single out-of-range
    row (only its 32-row unit recomputed): both equal the fp32 twin."""
    from paper_2412_04634_b200.mlp import full_forward, init_theta, make_spec

    spec = make_spec(depth=2)
    th = init_theta(spec, seed=1, out_scale=0.1)
    q = O.measure_queries(5000, seed=3)
    w0 = int(spec.w_off[0])
    big = th.copy()
    big[w0 + 5] = 7.0e4  # one weight beyond fp16
    big[int(spec.w_off[-1]):] *= np.float32(1e-4)
    y2 = full_forward(spec, big, *q, precision=2)
    y1 = full_forward(spec, big, *q, precision=1)
    np.testing.assert_allclose(y2, y1, rtol=1e-5, atol=1e-9)
    # 64 hash slots of the finest level blown up to 1e5: only the ~1.6 % of
    # rows that gather one of them (and their 32-row units) are recomputed
    hot = th.copy()
    l11 = 11 * spec.table * spec.feats
    hot[l11: l11 + 128] = np.float32(1e5)
    y2 = full_forward(spec, hot, *q, precision=2)
    y1 = full_forward(spec, hot, *q, precision=1)
    np.testing.assert_allclose(y2, y1, rtol=1e-4, atol=1e-7 * float(np.abs(y1).max()))


def test_non_finite_theta_raises(nb):
    """mlp.py:104-105: full_forward / query raise DivergenceError on a
    non-finite theta -- the fused kernels check it on the device."""
    from paper_2412_04634_b200.errors import DivergenceError
    from paper_2412_04634_b200.mlp import full_forward, init_theta, make_spec, query

    spec = make_spec(depth=2)
    th = init_theta(spec, seed=1, out_scale=0.1)
    q = O.measure_queries(300, seed=2)
    for bad_at in (17, int(spec.w_off[1]) + 3):
        t = th.copy()
        t[bad_at] = np.nan
        for prec in (0, 1, 2):
            with pytest.raises(DivergenceError):
                full_forward(spec, t, *q, precision=prec)
        surf = np.concatenate([q[0], q[1], q[2], q[3][:, None]], axis=1)[:10]
        with pytest.raises(DivergenceError):
            query(spec, t, surf, q[4], np.arange(300, dtype=np.int32) % 10)
    # pinned host tensors take the copy/compute pipeline: same check
    pinned = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in q]
    t = th.copy()
    t[3] = np.inf
    with pytest.raises(DivergenceError):
        full_forward(spec, t, *pinned)


def test_pinned_pipeline_matches_device_path(nb):
    """The pinned-host copy/compute/copy pipeline (the e2e path) returns a
    complete, synchronised host result equal to the device-resident call."""
    from paper_2412_04634_b200 import mlp

    spec = mlp.make_spec(depth=2)
    th = torch.from_numpy(mlp.init_theta(spec, seed=1, out_scale=0.1)).cuda()
    n = 3 * (1 << 19) + 777  # several chunks plus a ragged tail
    q = O.measure_queries(n, seed=9)
    pinned = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in q]
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in q]
    y_pipe = mlp.full_forward(spec, th, *pinned)
    assert not y_pipe.is_cuda
    y_host = y_pipe.numpy().copy()  # read immediately: must already be complete
    y_dev = mlp.full_forward(spec, th, *dev).cpu().numpy()
    assert np.array_equal(y_host, y_dev)


def test_numpy_staged_path_matches_device_path(nb):
    """Large numpy batches (the reference's types) stream through pinned
    staging with overlapped copies: a fresh numpy result equal to the
    device-resident call, over several chunks and a ragged tail."""
    from paper_2412_04634_b200 import mlp

    spec = mlp.make_spec(depth=2)
    th_np = mlp.init_theta(spec, seed=1, out_scale=0.1)
    n = 3 * (1 << 18) + 555
    q = [np.ascontiguousarray(a) for a in O.measure_queries(n, seed=4)]
    y_np = mlp.full_forward(spec, th_np, *q)  # >= 2^18 rows: the staged path
    assert isinstance(y_np, np.ndarray) and y_np.shape == (n, 3)
    th = torch.from_numpy(th_np).cuda()
    dev = [torch.from_numpy(a).cuda() for a in q]
    y_dev = mlp.full_forward(spec, th, *dev).cpu().numpy()
    assert np.array_equal(y_np, y_dev)
    y_small = mlp._full_forward_numpy(spec, th, q, 2, chunk=1 << 16)  # many chunks
    assert np.array_equal(y_small, y_dev)


def test_query_amortised_bad_index_async(nb):
    """nirc_query encodes each surface once; a bad surface index is reported
    through the device status word (ConfigError at the result read) and the
    good rows still equal full_forward on the gathered rows."""
    from paper_2412_04634_b200.errors import ConfigError
    from paper_2412_04634_b200.mlp import full_forward, init_theta, make_spec, query

    spec = make_spec(depth=4)
    th = init_theta(spec, seed=4, out_scale=0.2)
    rng = np.random.default_rng(1)
    ns_ = 500
    nrm = rng.normal(size=(ns_, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    surf = np.concatenate([rng.uniform(size=(ns_, 3)), nrm, rng.uniform(size=(ns_, 3)),
                           rng.uniform(size=(ns_, 1))], axis=1)
    n = 17 * ns_
    idx = np.repeat(np.arange(ns_, dtype=np.int32), 17)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    for prec in (1, 2):
        y = query(spec, th, surf, d, idx, precision=prec)
        s = surf[idx]
        y2 = full_forward(spec, th, s[:, 0:3], s[:, 3:6], s[:, 6:9], s[:, 9], d, precision=prec)
        np.testing.assert_array_equal(y, np.asarray(y2))
    bad = idx.copy()
    bad[1234] = -1
    with pytest.raises(ConfigError):
        query(spec, th, surf, d, bad)


@pytest.mark.parametrize("tag,depth", [("corn", 2), ("bright", 4)])
def test_two_level_render_trained_cache(nb, golden, tag, depth):
    """render_two_level with the reference-trained cache (64^2, nc=(8,),
    1 spp, frame = the cache's frame) against the reference's image."""
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.estimators import EstimatorConfig, render
    from paper_2412_04634_b200.scene import load_scene

    import scene_texts as T

    g = golden("trained")
    sc = load_scene(T.corn_text(64, 100.0 if tag == "bright" else 1.0))
    cache = Cache.create("nirc", sc, seed=5, depth=depth)
    cache.theta.copy_(torch.from_numpy(g[f"{tag}_theta"]))
    for prec in (0, 2):
        r = render(sc, EstimatorConfig(mode="two-level", nc=(8,), max_cache_vertices=1),
                   cache=cache, seed=3, spp=1, frame=int(g[f"{tag}_frame"]), precision=prec)
        assert np.array_equal(r.path_length, g[f"{tag}_tl_plen"])
        ref = g[f"{tag}_tl_image"]
        np.testing.assert_allclose(r.image, ref, rtol=1e-5, atol=5e-7 * max(1.0, ref.max() / 17))


@pytest.mark.parametrize("nc", [8, 16])  # nc = 16: the warp-specialised kernel (k_infer_ws)
def test_render_fp16_range_guard(nb, golden, nc):
    """The range-stress net in the two-level frame: the 2xFP16 inference
    kernel flags the tiles and k_infer_fix recomputes them; the image
    equals the 3xTF32 render (fp32 range) to the network tolerance."""
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.estimators import EstimatorConfig, render
    from paper_2412_04634_b200.scene import load_scene

    import scene_texts as T

    g = golden("trained")
    sc = load_scene(T.corn_text(64))
    cache = Cache.create("nirc", sc, seed=5, depth=2)
    spec = cache.spec
    th = g["corn_theta"].copy()
    s = np.float32(float(g["stress_theta_scale"]))
    th[int(spec.w_off[0]): int(spec.b_off[0]) + int(spec.dims[1])] *= s
    th[int(spec.w_off[-1]):] *= np.float32(1.0) / s
    cache.theta.copy_(torch.from_numpy(th))
    cfg = EstimatorConfig(mode="two-level", nc=(nc,), max_cache_vertices=1)
    r2 = render(sc, cfg, cache=cache, seed=3, spp=1, precision=2)
    r0 = render(sc, cfg, cache=cache, seed=3, spp=1, precision=0)
    assert np.all(np.isfinite(r2.image))
    np.testing.assert_allclose(r2.image, r0.image, rtol=1e-5, atol=5e-7)


@pytest.mark.parametrize("nc", [8, 16])
def test_concurrent_renders_on_two_streams(nb, nc):
    """parameters are read-only snapshots, callable
    concurrently: two caches with different theta render (and run the fused
    forward) at the same time on two streams, device-resident, no host sync
    in between; each result equals its serial run bit for bit (the packed
    weight image is per call, not library state)."""
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.estimators import EstimatorConfig, render_device
    from paper_2412_04634_b200.mlp import full_forward
    from paper_2412_04634_b200.scene import load_builtin

    sc = load_builtin("cornell").with_resolution(96, 96)
    c1 = Cache.create("nirc", sc, seed=1, init="random")
    c2 = Cache.create("nirc", sc, seed=2, init="random")
    c2.theta.mul_(1.5)
    cfg = EstimatorConfig(mode="two-level", nc=(nc,), max_cache_vertices=1)
    q = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in O.measure_queries(1 << 16, 5)]

    def run(c):
        img = render_device(sc, cfg, cache=c, seed=4, spp=2)[0]
        return img, full_forward(c.spec, c.theta, *q)

    ser = [[t.cpu().numpy() for t in run(c)] for c in (c1, c2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for rep in range(3):
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            r1 = run(c1)
        with torch.cuda.stream(s2):
            r2 = run(c2)
        torch.cuda.synchronize()
        for got, want in ((r1, ser[0]), (r2, ser[1])):
            for a, b in zip(got, want):
                assert np.array_equal(a.cpu().numpy(), b), rep


@pytest.mark.parametrize("depth,nc", [(2, (16,)), (4, (16,)), (2, (4,)), (2, (6, 5, 1))])
def test_warp_specialised_inference_matches_grouped_kernel(nb, depth, nc, monkeypatch):
    """k_infer_ws (producer warpgroups + four chain groups, the default for
    nc >= 8 where its shared-memory plan fits) against the grouped k_infer_tc
    (NIRC_INFER_NP=0) on the same frame: same walks, the same deferred
    vertices and pixels within the two splits' rounding."""
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.estimators import EstimatorConfig, render

    sc = __import__("paper_2412_04634_b200.scene", fromlist=["load_builtin"]).load_builtin(
        "cornell").with_resolution(128, 96)
    cache = Cache.create("nirc", sc, seed=7, init="random", depth=depth)
    # nc = (4,): 25 vertices per tile, the producers' encoding pass runs
    # three rounds; (6, 5, 1): 18 per tile, three cache vertices per path
    # (both fit k_infer_ws's shared-memory plan at depth 2)
    cfg = EstimatorConfig(mode="two-level", nc=nc, max_cache_vertices=len(nc))
    ws = render(sc, cfg, cache=cache, seed=2, spp=2, precision=2)
    # the configuration runs k_infer_ws: its timing ablation (chains skip
    # their MMAs, tools only) changes the image
    monkeypatch.setenv("NIRC_INFER_ABLATE", "2")
    ablated = render(sc, cfg, cache=cache, seed=2, spp=2, precision=2)
    assert not np.array_equal(ablated.image, ws.image)
    monkeypatch.delenv("NIRC_INFER_ABLATE")
    monkeypatch.setenv("NIRC_INFER_NP", "0")
    grouped = render(sc, cfg, cache=cache, seed=2, spp=2, precision=2)
    assert np.array_equal(ws.path_length, grouped.path_length)
    assert ws.queries == grouped.queries > 0
    np.testing.assert_allclose(ws.image, grouped.image, rtol=1e-5, atol=1e-7)
