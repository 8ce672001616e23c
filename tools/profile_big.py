"""One warm-up and one profiled 1080p PT frame of the larger test scene
(tests/big_scene.py) for ncu."""
import os
import sys

_ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path[:0] = [_ROOT, os.path.join(_ROOT, "tests")]
import torch  # noqa: E402
from big_scene import big_scene_text  # noqa: E402

from paper_2412_04634_b200.estimators import EstimatorConfig, render_device  # noqa: E402
from paper_2412_04634_b200.scene import load_scene  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
sc = load_scene(big_scene_text(nq, max(1, nq // 30))).with_resolution(1920, 1080)
for f in range(2):
    render_device(sc, EstimatorConfig(mode="pt"), None, 0, 1, f)
torch.cuda.synchronize()
