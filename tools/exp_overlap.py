"""1080p cfg3 frames: sequential run_frame vs FramePipeline (render || train)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2412_04634_b200.caches import Cache  # noqa: E402
from paper_2412_04634_b200.frame import FramePipeline, config3, run_frame  # noqa: E402
from paper_2412_04634_b200.scene import load_builtin  # noqa: E402

for mode in ("seq", "pipe", "seq", "pipe"):
    scene = load_builtin("cornell").with_resolution(1920, 1080)
    cache = Cache.create("nirc", scene, seed=0, init="random")
    cfg = config3((16,))
    pipe = FramePipeline(scene, cache, cfg, seed=0) if mode == "pipe" else None
    ts = []
    for f in range(13):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if pipe:
            pipe.step(f)
        else:
            run_frame(scene, cache, cfg, 0, f)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    ts = sorted(ts[3:])
    print(mode, "median ms", round(ts[len(ts) // 2], 3), "min", round(ts[0], 3))
