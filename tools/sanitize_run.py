"""Small launches of every hand-written tensor-core / tracer kernel, sized for
compute-sanitizer (memcheck / racecheck / synccheck run each launch 10-100x
slower):

  k_full_forward_tc (F16x2 TS chain and 3xTF32), k_infer_tc (two-level frame),
  k_trace (+ record walks), the training kernels (k_train_tc / k_train_tile,
  selection, scatter, Adam), and the f64 shadow path.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
Prints "sanitize workload ok" at the end."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import nirc_oracle as O  # noqa: E402
from paper_2412_04634_b200.caches import Cache, train_frame  # noqa: E402
from paper_2412_04634_b200.estimators import EstimatorConfig, render_and_collect  # noqa: E402
from paper_2412_04634_b200.mlp import full_forward, init_theta, make_spec  # noqa: E402
from paper_2412_04634_b200.scene import load_builtin  # noqa: E402

which = set(sys.argv[1:]) or {"forward", "frame", "train"}
torch.cuda.set_device(0)
if "forward" in which:
    spec = make_spec(depth=2)
    theta = init_theta(spec, seed=1, out_scale=0.1)
    q = O.measure_queries(3000, seed=3)
    for prec in (2, 0):
        y = full_forward(spec, theta, *q, precision=prec)
        assert np.all(np.isfinite(y))
    spec4 = make_spec(depth=4)
    y = full_forward(spec4, init_theta(spec4, seed=2, out_scale=0.1), *q)
    print("forward ok", flush=True)
if "frame" in which or "train" in which:
    sc = load_builtin("cornell").with_resolution(48, 32)
    cache = Cache.create("nirc", sc, seed=2, init="random")
    cfg = EstimatorConfig(mode="two-level", nc=(16,), max_cache_vertices=1)
    img, img2, term, queries, rec = render_and_collect(sc, cfg, cache, seed=1, spp=1, frame=0,
                                                       count=2048)
    torch.cuda.synchronize()
    print("frame ok", int(queries.item()), len(rec), flush=True)
    if "train" in which:
        trace = train_frame(cache, rec, steps=2, batch=1024)
        torch.cuda.synchronize()
        print("train ok", trace, flush=True)
print("sanitize workload ok", flush=True)
