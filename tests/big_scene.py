"""A larger test scene: the BOX room plus a field
of small tilted quads and spheres -- past HOST_BVH_MAX, so the scene's BVH
is built on the device.  Deterministic text; shared by the golden generator
(tests/golden/make_golden.py big) and the tests."""

import numpy as np

ROOM = """
camera { position 0.5 0.5 -1.4  look_at 0.5 0.5 0.5  up 0 1 0
         fov 39  resolution 16 16 }
material w { kind lambert  albedo 0.7 0.7 0.7 }
material r { kind lambert  albedo 0.6 0.2 0.1 }
material g { kind conductor  albedo 0.9 0.6 0.3  roughness 0.3 }
material l { kind lambert  albedo 0 0 0  emit 10 10 10 }
quad floor   { material w  p0 0 0 0  p1 1 0 0  p2 1 0 1  p3 0 0 1 }
quad ceiling { material w  p0 0 1 0  p1 0 1 1  p2 1 1 1  p3 1 1 0 }
quad back    { material w  p0 0 0 1  p1 1 0 1  p2 1 1 1  p3 0 1 1 }
quad left    { material w  p0 0 0 0  p1 0 0 1  p2 0 1 1  p3 0 1 0 }
quad right   { material w  p0 1 0 0  p1 1 1 0  p2 1 1 1  p3 1 0 1 }
quad lamp    { material l  p0 0.35 0.999 0.35  p1 0.65 0.999 0.35
               p2 0.65 0.999 0.65  p3 0.35 0.999 0.65 }
"""


def big_scene_text(n_quads=1200, n_spheres=40, seed=7):
    rng = np.random.default_rng(seed)
    lines = [ROOM]
    for i in range(n_quads):
        c = rng.uniform(0.05, 0.95, 3)
        c[1] = rng.uniform(0.02, 0.6)
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        v = np.cross(u, rng.normal(size=3))
        v /= np.linalg.norm(v)
        s = rng.uniform(0.005, 0.03)
        p = [c - s * u - s * v, c + s * u - s * v, c + s * u + s * v, c - s * u + s * v]
        mat = "wrg"[i % 3]
        pts = "  ".join(f"p{k} {float(q[0])!r} {float(q[1])!r} {float(q[2])!r}"
                        for k, q in enumerate(p))
        lines.append(f"quad q{i} {{ material {mat}  {pts} }}")
    for i in range(n_spheres):
        c = rng.uniform(0.1, 0.9, 3)
        c[1] = rng.uniform(0.05, 0.5)
        r = rng.uniform(0.01, 0.04)
        cs = " ".join(repr(float(x)) for x in c)
        lines.append(f"sphere s{i} {{ material {'wg'[i % 2]}  center {cs}  radius {float(r)!r} }}")
    return "\n".join(lines) + "\n"
