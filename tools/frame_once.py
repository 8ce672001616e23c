"""One 1080p two-level Cornell frame (cfg3 render path, nc=(16,)) after one
warm-up -- the command profiled by ncu for the inference kernel."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
import torch  # noqa: E402

from paper_2412_04634_b200.caches import Cache  # noqa: E402
from paper_2412_04634_b200.estimators import EstimatorConfig, render_device  # noqa: E402
from paper_2412_04634_b200.scene import load_builtin  # noqa: E402

w, h = (int(x) for x in os.environ.get("RES", "1920x1080").split("x"))
sc = load_builtin("cornell").with_resolution(w, h)
cache = Cache.create("nirc", sc, seed=1, init="random")
cfg = EstimatorConfig(mode="two-level", nc=(16,), max_cache_vertices=1)
for _ in range(2):
    render_device(sc, cfg, cache=cache, seed=0, spp=1)
torch.cuda.synchronize()
