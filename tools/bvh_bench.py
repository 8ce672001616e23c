"""Device BVH build vs the host restatement on primitive soups, and a 1080p
PT / two-level frame on the larger test scene family.
Prints one JSON line per measurement."""
import json
import os
import sys
import time

import numpy as np
import torch

_ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path[:0] = [_ROOT, os.path.join(_ROOT, "tests")]
from big_scene import big_scene_text  # noqa: E402

from paper_2412_04634_b200 import scene as S  # noqa: E402


def soup(n, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, (n, 3)), rng.normal(0, 0.01, (n, 3)), rng.normal(0, 0.01, (n, 3)),
            np.zeros((0, 3)), np.zeros(0))


for n in (10_000, 100_000, 1_000_000, 4_000_000):
    a = soup(n)
    S.build_bvh_device(*a)  # warm (CUB temp sizing, module load)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        S.build_bvh_device(*a)
    dev_s = (time.perf_counter() - t) / 3
    host_s = None
    if n <= 100_000:
        t = time.perf_counter()
        S.build_bvh(*a)
        host_s = time.perf_counter() - t
    print(json.dumps({"bvh_build": n, "device_ms": round(dev_s * 1e3, 2),
                      "host_ms": None if host_s is None else round(host_s * 1e3, 1)}))

from paper_2412_04634_b200.caches import Cache  # noqa: E402
from paper_2412_04634_b200.estimators import EstimatorConfig, render_device  # noqa: E402

for nq in (1200, 20000):
    sc = S.load_scene(big_scene_text(nq, nq // 30)).with_resolution(1920, 1080)
    nprim = len(sc.pack.tri_v0) + len(sc.pack.sph_c)
    cache = Cache.create("nirc", sc, seed=9, init="random")
    for mode, cfg, c in (("pt", EstimatorConfig(mode="pt"), None),
                         ("two-level", EstimatorConfig(mode="two-level", nc=(16,),
                                                       max_cache_vertices=1), cache)):
        for _ in range(2):
            render_device(sc, cfg, c, seed=0, spp=1, frame=0, force_cache=c is not None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for f in range(5):
            render_device(sc, cfg, c, seed=0, spp=1, frame=f, force_cache=c is not None)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"scene_prims": nprim, "mode": mode, "res": "1920x1080",
                          "ms_per_frame": round(e0.elapsed_time(e1) / 5, 3)}))
