"""Host-side pieces of the drop-in API (no GPU): scene parsing and the flat
pack (bit-identical to the reference's ScnPack, pinned by sha1 digests the
reference produced), snapshots, rng, configuration validation."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

BOX = open(os.path.join(GOLDEN, "make_golden.py")).read().split('BOX = """')[1].split('"""')[0]
MIXED = open(os.path.join(GOLDEN, "make_golden.py")).read().split('MIXED = """')[1].split('"""')[0]


def _scenes():
    from paper_2412_04634_b200.scene import load_builtin, load_scene

    s = {n: load_builtin(n) for n in ("cornell", "furnace", "occlusion", "teleport")}
    s["teleport@50"] = load_builtin("teleport").at_frame(50)
    s["BOX"] = load_scene(BOX)
    s["MIXED"] = load_scene(MIXED)
    return s


def test_scene_packs_bit_identical_to_reference():
    ref = json.load(open(os.path.join(GOLDEN, "scene_packs.json")))
    for name, sc in _scenes().items():
        for f in sc.pack._fields:
            a = np.ascontiguousarray(np.asarray(getattr(sc.pack, f)))
            dt, shape, digest = ref[name][f]
            assert (str(a.dtype), list(a.shape)) == (dt, shape), (name, f)
            assert hashlib.sha1(a.tobytes()).hexdigest() == digest, (name, f)
        assert hashlib.sha1(np.asarray(sc.camera).tobytes()).hexdigest() == ref[name]["camera"]


def test_parse_errors():
    from paper_2412_04634_b200.errors import ConfigError, ParseError
    from paper_2412_04634_b200.scene import load_scene

    with pytest.raises(ParseError):
        load_scene("camera { fov 40 } bogus { }")
    with pytest.raises(ParseError):
        load_scene("material m { kind plastic }\ncamera { }")
    with pytest.raises(ParseError):
        load_scene("camera { }\nquad q { material nope p0 0 0 0 p1 1 0 0 p2 1 1 0 p3 0 1 0 }")
    with pytest.raises(ParseError):
        load_scene("material m { kind lambert }")  # no camera
    with pytest.raises(ConfigError):
        load_scene("camera { }\nmaterial m { kind lambert }\n"
                   "tri t { material m p0 0 0 0 p1 1 1 1 p2 2 2 2 }")  # degenerate


def test_host_intersect_matches_reference_convention():
    from paper_2412_04634_b200.scene import load_scene

    sc = load_scene(BOX)
    it = sc.intersect([0.5, 0.5, 0.5], [0.0, -1.0, 0.0])
    assert it is not None and abs(it.position[1]) < 1e-12
    assert np.allclose(it.ns, [0.0, 1.0, 0.0])
    assert sc.intersect([0.5, 0.5, 0.5], [0.0, 0.0, -1.0]) is None  # open front


def test_snapshot_roundtrip_and_errors(tmp_path):
    from paper_2412_04634_b200.errors import ConfigError
    from paper_2412_04634_b200.snapshot import load_snapshot, save_snapshot

    p = str(tmp_path / "s.bin")
    data = {"theta": np.arange(10, dtype=np.float32), "m": np.ones((2, 3)),
            "step": np.int64(42), "u": np.arange(3, dtype=np.uint64),
            "i": np.arange(4, dtype=np.int32)}
    save_snapshot(p, data)
    out = load_snapshot(p)
    for k, v in data.items():
        assert np.array_equal(out[k], v) and out[k].dtype == np.asarray(v).dtype
    assert out["step"].shape == ()
    bad = tmp_path / "junk"
    bad.write_bytes(b"NOPE" * 4)
    with pytest.raises(ConfigError):
        load_snapshot(str(bad))
    blob = open(p, "rb").read()
    (tmp_path / "t").write_bytes(blob[:-20])
    with pytest.raises(ConfigError):
        load_snapshot(str(tmp_path / "t"))


def test_estimator_config_validation():
    from paper_2412_04634_b200.errors import ConfigError
    from paper_2412_04634_b200.estimators import EstimatorConfig

    EstimatorConfig(mode="two-level", nc=(28,), max_cache_vertices=1)
    for bad in (dict(mode="nope"), dict(nc=(29, 1, 1)), dict(nr=2), dict(rr=1.0),
                dict(nc=(1,), max_cache_vertices=2), dict(sph_c=0.0)):
        with pytest.raises(ConfigError):
            EstimatorConfig(**bad)


def test_rng_host_matches_oracle():
    import nirc_oracle as O

    from paper_2412_04634_b200 import rng

    for args in ((0, 4, 3, 100, 0), (7, 2, 5, 1000, 17)):
        assert np.array_equal(rng.uniform_array(*args), O.uniform_array(*args))
        assert np.array_equal(rng.normal_array(*args), O.normal_array(*args))
    assert rng.stream_key(5, 1, 3, 77, 1) == O.stream_key(5, 1, 3, 77, 1)


def test_make_spec_and_init_theta_match_oracle():
    import nirc_oracle as O

    from paper_2412_04634_b200.mlp import init_theta, make_spec

    for depth in (2, 4):
        s = make_spec(depth=depth)
        o = O.Spec(depth=depth)
        assert s.theta_len == o.theta_len and list(s.w_off) == o.w_off
        assert np.array_equal(s.res, o.res)
        assert np.array_equal(init_theta(s, seed=1, out_scale=0.1),
                              O.init_theta(o, seed=1, out_scale=0.1))
    assert make_spec().in_dim == 47 and make_spec().theta_len == 802179


def test_reference_snapshots_roundtrip_bytes():
    """NNCACHE1 files written by the reference's Cache.save parse with the
    host reader and re-serialise byte for byte (snapshot.py:31-77)."""
    from paper_2412_04634_b200.snapshot import load_snapshot, save_snapshot

    for name in ("snapshot_fresh", "snapshot_trained"):
        path = os.path.join(GOLDEN, name + ".nncache")
        d = load_snapshot(path)
        assert {"theta", "m", "v", "t", "frame", "net", "bb_min", "bb_ext"} <= set(d)
        import tempfile

        with tempfile.TemporaryDirectory() as td:
            out = os.path.join(td, "x.nncache")
            save_snapshot(out, d)
            assert open(out, "rb").read() == open(path, "rb").read(), name
    t = load_snapshot(os.path.join(GOLDEN, "snapshot_trained.nncache"))
    assert int(t["t"]) == 2 and int(t["frame"]) == 1 and np.any(t["m"] != 0)
