"""Wall time of the drop-in run_experiment (experiment.py:122-213) on the
teleport scene at 1080p, 100 frames, ref_spp 64."""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2412_04634_b200.config import RunConfig  # noqa: E402
from paper_2412_04634_b200.experiment import run_experiment  # noqa: E402
from paper_2412_04634_b200.scene import load_builtin  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 100
with tempfile.TemporaryDirectory() as d:
    cfg = RunConfig(scene="teleport", mode="two-level", nc=(16,), max_cache_vertices=1,
                    frames=frames, seed=0, out=os.path.join(d, "o"), ref_dir=os.path.join(d, "r"),
                    ref_spp=64)
    t = time.perf_counter()
    out = run_experiment(cfg, scene=load_builtin("teleport").with_resolution(1920, 1080))
    dt = time.perf_counter() - t
print({"frames": frames, "wall_s": round(dt, 3), "ms_per_frame": round(dt / frames * 1e3, 2),
       "mrse_first": round(out.rows[0]["mrse"], 4), "mrse_last": round(out.rows[-1]["mrse"], 4)})
