"""First mismatches of the fast intersect paths vs the reference-order walk."""
import ctypes as C
import os
import sys

_ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path[:0] = [_ROOT, os.path.join(_ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
from big_scene import big_scene_text  # noqa: E402

from paper_2412_04634_b200 import _lib  # noqa: E402
from paper_2412_04634_b200.scene import load_scene  # noqa: E402

src = open(os.path.join(_ROOT, "tests", "golden", "make_golden.py")).read()
MIXED = src.split('MIXED = """')[1].split('"""')[0]
lib = _lib.load()
fn = lib.nirc_debug_intersect_detail
fn.argtypes = [C.POINTER(_lib.NircScene), C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p,
               C.c_int32]
np.set_printoptions(precision=17, linewidth=200)
for (name, text), aim in [(x, a) for x in (("mixed", MIXED), ("big", big_scene_text()))
                          for a in (1, 0)]:
    ds = load_scene(text).device()
    counts = torch.zeros((2,), dtype=torch.int64, device="cuda")
    det = torch.zeros((16, 16), dtype=torch.float64, device="cuda")
    fn(ds.ptr(), 1 << 22, 321, C.c_void_p(counts.data_ptr()), C.c_void_p(det.data_ptr()), aim)
    torch.cuda.synchronize()
    print(name, "aimed" if aim else "random", counts.tolist())
    for r in det.cpu().numpy()[:6]:
        print(" fast", r[6:9], "ref", r[9:12], "occ", r[12:16])
