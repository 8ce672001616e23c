"""Timeline of the four chain groups of k_infer_ws in CTA 0 (cfg3 frame):
per tile and layer, the elected thread's MMA issue start / end and the
completion seen by warp 0.  Prints per-layer medians and how much of the time
at least one group has MMAs outstanding (an upper bound of the tensor pipe's
busy time) and how many groups overlap."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_04634_b200 import _lib  # noqa: E402
from paper_2412_04634_b200.caches import Cache  # noqa: E402
from paper_2412_04634_b200.estimators import render_device  # noqa: E402
from paper_2412_04634_b200.frame import config3  # noqa: E402
from paper_2412_04634_b200.scene import load_builtin  # noqa: E402

lib = _lib.load()
buf = torch.zeros(16384, dtype=torch.int64, device="cuda")
sc = load_builtin("cornell").with_resolution(1920, 1080)
cache = Cache.create("nirc", sc, seed=0, init="random")
cfg = config3()
render_device(sc, cfg, cache)
lib.nirc_debug_infer_probe(C.c_void_p(buf.data_ptr()))
render_device(sc, cfg, cache)
torch.cuda.synchronize()
lib.nirc_debug_infer_probe(None)
a = buf.cpu().numpy()[4096:4096 + 4 * 512].reshape(4, 32, 16).astype(np.float64)
NL = 5
iv = []  # (start, end, group) of MMA windows
issue, window = [[] for _ in range(NL)], [[] for _ in range(NL)]
for g in range(4):
    for n in range(4, 28):
        t = a[g, n]
        if t[0] == 0 or t[3 * (NL - 1) + 2] == 0:
            continue
        for l in range(NL):
            s, e, d = t[3 * l], t[3 * l + 1], t[3 * l + 2]
            if s and e and d:
                issue[l].append(e - s)
                window[l].append(d - s)
                iv.append((s, d, g))
print("per layer: issue cycles (median), issue->done cycles (median)")
for l in range(NL):
    print(f"  layer {l}: {np.median(issue[l]):7.0f} {np.median(window[l]):7.0f}")
iv.sort()
lo = min(x[0] for x in iv)
hi = max(x[1] for x in iv)
ev = sorted([(s, 1) for s, _, _ in iv] + [(d, -1) for _, d, _ in iv])
busy = {k: 0.0 for k in range(5)}
cur, last = 0, ev[0][0]
for t, dlt in ev:
    busy[min(cur, 4)] += t - last
    cur += dlt
    last = t
tot = hi - lo
print(f"span {tot:.0f} cycles; fraction of time with k groups' MMAs outstanding:",
      {k: round(v / tot, 3) for k, v in busy.items()})
g0 = a[0, 8]
print("group 0 tile 8 (relative cycles):", [int(x - g0[0]) if x else None for x in g0[:15]])
# producer 0 of CTA 0: per tile [start, records ready, encoding done, rows
# built + slot free, arrive] (infer_ws.cuh probes pb[0..4])
pr = buf.cpu().numpy()[2048:2048 + 32 * 8].reshape(32, 8).astype(np.float64)
ok = [t for t in pr[2:] if t[0] and t[4]]
if ok:
    d = np.array([[t[1] - t[0], t[2] - t[1], t[5] - t[2], t[6] - t[5], t[3] - t[6], t[4] - t[3]]
                  for t in ok])
    per = np.diff([t[0] for t in ok])
    print("  of the records phase, issuing the next tile's copies: %.0f"
          % np.median([t[7] - t[0] for t in ok]))
    print("producer 0 phases (median cycles): records %.0f, encoding %.0f, vertex chunks %.0f, "
          "rows %.0f, slot wait %.0f, stores + meta %.0f; tile interval %.0f"
          % (*np.median(d, axis=0), np.median(per)))
