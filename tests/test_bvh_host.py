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


def test_scan_items_cover_each_triangle_once():
    """devscene.filter_items (the warp-uniform scan's pre-test items): every
    scan-order triangle is covered by exactly one item; quads split along a
    shared diagonal become parallelogram items (cu = 0) whose edges are the
    two outer edges of the pair, triangles left over stay triangles."""
    from paper_2412_04634_b200.devscene import filter_items
    from paper_2412_04634_b200.scene import load_builtin

    for name, n_items in (("cornell", 18), ("teleport", 6), ("occlusion", 2)):
        p = load_builtin(name).pack
        items = filter_items(p)
        assert items.shape == (n_items, 16)
        masks = items[:, 14:16].copy().view(np.uint32).astype(np.uint64)
        bits = masks[:, 0] | (masks[:, 1] << np.uint64(32))
        total = np.uint64(0)
        for b in bits:
            assert (total & b) == 0
            total |= b
        n = len(p.tri_v0)
        assert int(total) == (1 << n) - 1
        for row, b in zip(items, bits):
            paired = bin(int(b)).count("1") == 2
            assert (row[12] == 0.0) == paired
            if paired:  # v0 + u e1 + v e2 over the unit square spans both triangles
                k1, k2 = [k for k in range(n) if int(b) >> k & 1]
                order = np.asarray(p.bvh_prim)
                e = {tuple(np.asarray(p.tri_e1)[order[k]]) for k in (k1, k2)} | \
                    {tuple(np.asarray(p.tri_e2)[order[k]]) for k in (k1, k2)}
                a_ = tuple(np.asarray(row[4:7], np.float64))
                assert any(np.allclose(a_, x, atol=1e-6) for x in e)
