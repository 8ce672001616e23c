"""FramePipeline (render(f) || train(f)) against the
sequential frame loop (frame.run_frame, experiment.py:149-185's order): path
lengths and record counts identical on every frame (the walks never read
theta), and -- the training being deterministic (fixed-point grid scatter,
fixed-order reductions) -- the same images and losses bit for bit on every
frame, including across the teleport scene's animation boundary."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(pipelined, frames, f0):
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.frame import FramePipeline, config3, run_frame
    from paper_2412_04634_b200.scene import load_builtin

    scene = load_builtin("teleport").with_resolution(96, 64)
    cache = Cache.create("nirc", scene, seed=3, init="random")
    cache.frame = f0
    cfg = config3((8,))
    pipe = FramePipeline(scene, cache, cfg, seed=1) if pipelined else None
    imgs, terms, stats = [], [], []
    for f in range(f0, f0 + frames):
        if pipelined:
            (img, _, term), st = pipe.step(f)
        else:
            sc = scene.at_frame(f)
            cache.scene = sc
            (img, _, term), st = run_frame(sc, cache, cfg, 1, f)
        torch.cuda.synchronize()
        imgs.append(img.cpu().numpy())
        terms.append(term.cpu().numpy())
        stats.append(st)
    return imgs, terms, stats, cache.theta.cpu().numpy()


def test_pipeline_matches_sequential_frames():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    # frames 37..42 cross the lamp jump at frame 40
    a = _run(False, 6, 37)
    b = _run(True, 6, 37)
    for f in range(6):
        assert np.array_equal(a[1][f], b[1][f]), f          # path lengths
        assert a[2][f].records == b[2][f].records, f
        assert a[2][f].queries == b[2][f].queries, f
    # frame 37 renders with the same initial theta: bit-identical
    assert np.array_equal(a[0][0], b[0][0])
    for f in range(1, 6):
        np.testing.assert_array_equal(b[0][f], a[0][f])
    la = np.array([s.loss for s in a[2]])
    lb = np.array([s.loss for s in b[2]])
    np.testing.assert_array_equal(lb, la)
    np.testing.assert_array_equal(b[3], a[3])  # the final theta
