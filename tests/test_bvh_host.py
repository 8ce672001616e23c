"""The host BVH restatement (scene.py build_bvh) against the reference's own
arrays for the larger scene (tests/golden/big.npz), and the C ABI's planned
node count (nirc_bvh_node_count, host-only) against the host build."""

import numpy as np

from big_scene import big_scene_text

KEYS = ("bvh_lo", "bvh_hi", "bvh_a", "bvh_b", "bvh_prim")


def test_host_bvh_matches_reference_on_big_scene(golden):
    from paper_2412_04634_b200 import scene as S

    desc = S.parse_scene(big_scene_text())
    sc = S.Scene.__new__(S.Scene)
    old = S.HOST_BVH_MAX
    S.HOST_BVH_MAX = 1 << 30  # force the host build here
    try:
        sc.__init__(desc, 0)
    finally:
        S.HOST_BVH_MAX = old
    g = golden("big")
    for k in KEYS:
        np.testing.assert_array_equal(getattr(sc.pack, k), g[k], err_msg=k)


def test_node_count_matches_host_build():
    from paper_2412_04634_b200 import _lib
    from paper_2412_04634_b200.scene import build_bvh

    lib = _lib.load()
    rng = np.random.default_rng(0)
    for n in (0, 1, 4, 5, 9, 63, 64, 65, 1000):
        v0 = rng.uniform(size=(n, 3))
        e = rng.uniform(size=(n, 3)) * 0.01
        nodes = len(build_bvh(v0, e, e[:, ::-1], np.zeros((0, 3)), np.zeros(0))[2])
        assert lib.nirc_bvh_node_count(n) == nodes
