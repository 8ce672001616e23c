"""cProfile of run_experiment (host overhead per frame)."""
import cProfile
import os
import pstats
import sys
import tempfile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2412_04634_b200.config import RunConfig  # noqa: E402
from paper_2412_04634_b200.experiment import run_experiment  # noqa: E402
from paper_2412_04634_b200.scene import load_builtin  # noqa: E402

with tempfile.TemporaryDirectory() as d:
    cfg = RunConfig(scene="teleport", mode="two-level", nc=(16,), max_cache_vertices=1,
                    frames=60, seed=0, out=os.path.join(d, "o"), ref_dir=os.path.join(d, "r"),
                    ref_spp=64)
    sc = load_builtin("teleport").with_resolution(1920, 1080)
    run_experiment(RunConfig(scene="teleport", mode="two-level", nc=(16,), max_cache_vertices=1,
                             frames=3, seed=0, out=os.path.join(d, "w"), ref_spp=4), scene=sc)
    pr = cProfile.Profile()
    pr.enable()
    run_experiment(cfg, scene=load_builtin("teleport").with_resolution(1920, 1080))
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
