"""1080p cfg3 render+collect: one launch set vs row bands on two streams
(band i's inference overlapping band i+1's trace)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2412_04634_b200.caches import Cache, default_train_count  # noqa: E402
from paper_2412_04634_b200.estimators import render_and_collect, render_device  # noqa: E402
from paper_2412_04634_b200.frame import config3  # noqa: E402
from paper_2412_04634_b200.scene import load_builtin  # noqa: E402

scene = load_builtin("cornell").with_resolution(1920, 1080)
cache = Cache.create("nirc", scene, seed=0, init="random")
cfg = config3((16,))
count = default_train_count(scene)
H = 1080
streams = [torch.cuda.current_stream(), torch.cuda.Stream()]
out = [torch.zeros((H, 1920, 3), dtype=torch.float64, device="cuda") for _ in range(2)]


def single(f):
    render_and_collect(scene, cfg, cache, 0, 1, f, count=count)


def banded(f, nb):
    cuts = [H * i // nb for i in range(nb + 1)]
    for i in range(nb):
        s = streams[i % 2]
        s.wait_stream(streams[0]) if i == 0 else None
        with torch.cuda.stream(s):
            if i == 0:
                render_and_collect(scene, cfg, cache, 0, 1, f, count=count,
                                   rows=(cuts[0], cuts[1]), defer=True)
            else:
                render_device(scene, cfg, cache, 0, 1, f, rows=(cuts[i], cuts[i + 1]))
    streams[0].wait_stream(streams[1])


for name, fn in (("single", single), ("bands2", lambda f: banded(f, 2)),
                 ("bands4", lambda f: banded(f, 4)), ("single", single),
                 ("bands3", lambda f: banded(f, 3)), ("bands6", lambda f: banded(f, 6))):
    ts = []
    for f in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        fn(f)
        e1.record(streams[0])
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    print(name, round(ts[len(ts) // 2], 3))
