import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from paper_2412_04634_b200.scene import load_scene
from paper_2412_04634_b200.estimators import pt_radiance, render, EstimatorConfig
src = open("tests/golden/make_golden.py").read()
BOX = src.split('BOX = """')[1].split('"""')[0]
box = load_scene(BOX)
g = np.load("tests/golden/api.npz")
for (ix, iy, s), want in zip(g["pix"], g["ptr"]):
    got = pt_radiance(box, int(ix), int(iy), seed=4, sample=int(s), frame=1)
    r = render(box, EstimatorConfig(mode="pt"), seed=4, spp=int(s) + 1, frame=1)
    print(ix, iy, s, "got", got, "want", want, "render mean*spp", r.image[iy, ix] * (s + 1))
