"""Dump the teleport convergence MRSE curve (tests/test_gpu_convergence.py's run)."""
import os, sys, tempfile
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2412_04634_b200.config import RunConfig
from paper_2412_04634_b200.experiment import run_experiment
from paper_2412_04634_b200.scene import load_builtin

g = np.load("tests/golden/convergence.npz")
frames, ref_spp, res = int(g["frames"]), int(g["ref_spp"]), int(g["res"])
with tempfile.TemporaryDirectory() as d:
    cfg = RunConfig(scene="teleport", mode="two-level", frames=frames, seed=0,
                    out=os.path.join(d, "out"), ref_dir=os.path.join(d, "ref"), ref_spp=ref_spp)
    out = run_experiment(cfg, scene=load_builtin("teleport").with_resolution(res, res))
m = np.array([r["mrse"] for r in out.rows])
np.save(sys.argv[1], m)
r = m / g["mrse"]
print(np.round(r, 3))
for lo, hi in ((30, 40), (40, 48), (54, 64), (8, 40), (40, 64), (1, 64)):
    print(lo, hi, round(m[lo:hi].mean() / g["mrse"][lo:hi].mean() - 1, 4))
