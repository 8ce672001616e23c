"""Per-phase cycle stamps of k_infer_tc (CTA 0, group 0) on a cfg3 frame."""
import ctypes as C
import os
import sys

os.environ.setdefault("NIRC_INFER_NP", "0")  # these stamps are k_infer_tc's (grouped kernel)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_04634_b200 import _lib  # noqa: E402
from paper_2412_04634_b200.caches import Cache  # noqa: E402
from paper_2412_04634_b200.estimators import render_device  # noqa: E402
from paper_2412_04634_b200.frame import config3  # noqa: E402
from paper_2412_04634_b200.scene import load_builtin  # noqa: E402

lib = _lib.load()
buf = torch.zeros(32 * 64, dtype=torch.int64, device="cuda")
sc = load_builtin("cornell").with_resolution(1920, 1080)
cache = Cache.create("nirc", sc, seed=0, init="random")
cfg = config3()
render_device(sc, cfg, cache)
lib.nirc_debug_infer_probe(C.c_void_p(buf.data_ptr()))
render_device(sc, cfg, cache)
torch.cuda.synchronize()
lib.nirc_debug_infer_probe(None)
a = buf.cpu().numpy().reshape(32, 64).astype(np.float64)
t = a[:, :5]
d = np.diff(t, axis=1)
tile = t[1:, 0] - t[:-1, 0]
print("phases (cycles): features, rows+A, chain, combine   | tile-to-tile")
print("median", np.median(d[2:30], axis=0).astype(int), int(np.median(tile[2:30])))
# chain detail: per layer  wait-for-MMA, then epilogue until next wait
ch = a[:, 5:15]
start = a[:, 2]
for i in range(3, 6):
    w = [ch[i, 2 * l + 1] - ch[i, 2 * l] for l in range(5)]
    e = [ch[i, 2 * (l + 1)] - ch[i, 2 * l + 1] for l in range(4)]
    print("tile", i, "to-first-wait", int(ch[i, 0] - start[i]), "mma-wait", [int(x) for x in w],
          "epilogue", [int(x) for x in e])

for i in range(3, 6):
    row = a[i]
    for l in range(3):
        w_end = row[5 + 2 * l + 1]
        e0, e1, e2 = row[21 + 3 * l], row[22 + 3 * l], row[23 + 3 * l]
        nxt = row[5 + 2 * (l + 1)]
        print(f"tile {i} layer {l}: ld+relu+split+sts {int(e0 - w_end)}  bias+fences {int(e1 - e0)}"
              f"  barrier {int(e2 - e1)}  issue {int(nxt - e2)}")

for i in range(3, 6):
    row = a[i]
    print("tile", i, "barrier->issue-start", [int(row[45 + 2 * l] - row[23 + 3 * l]) for l in range(3)],
          "issue 12 mma", [int(row[46 + 2 * l] - row[45 + 2 * l]) for l in range(3)],
          "after-issue->next wait", [int(row[5 + 2 * (l + 1)] - row[46 + 2 * l]) for l in range(3)])
