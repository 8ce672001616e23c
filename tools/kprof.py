"""Warm per-kernel device times with torch.profiler (CUPTI), no replay:
    python tools/kprof.py train      # 4-step cfg3-sized train_frame
    python tools/kprof.py frame      # 1080p two-level frame (cfg3)
Prints kernel name, calls, mean us, total us over the profiled iterations."""
import os
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402


def train_job():
    import nirc_oracle as O
    from paper_2412_04634_b200.adam import AdamState
    from paper_2412_04634_b200.caches import Records, train_frame_device
    from paper_2412_04634_b200.mlp import init_theta, make_spec

    n = int(os.environ.get("N_REC", 113895))
    spec = make_spec(depth=int(os.environ.get("DEPTH", 4)))
    r = O.synth_records(n, seed=3)
    rec = Records(kind="nirc", frame=0, n=n,
                  **{k: torch.as_tensor(v).cuda() for k, v in r.items()})
    theta = torch.from_numpy(init_theta(spec, seed=1, out_scale=0.1)).cuda()
    adam = AdamState(theta)
    det = os.environ.get("DET", "0") == "1"
    return lambda: train_frame_device(spec, theta, rec, seed=0, frame=0, steps=4, adam=adam,
                                      deterministic=det)


def frame_job():
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.estimators import EstimatorConfig, render_device
    from paper_2412_04634_b200.scene import load_builtin

    sc = load_builtin("cornell").with_resolution(1920, 1080)
    cache = Cache.create("nirc", sc, seed=1, init="random")
    cfg = EstimatorConfig(mode="two-level", nc=(16,), max_cache_vertices=1)
    return lambda: render_device(sc, cfg, cache=cache, seed=0, spp=1)


job = {"train": train_job, "frame": frame_job}[sys.argv[1]]()
iters = int(os.environ.get("ITERS", 5))
for _ in range(3):
    job()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(iters):
        job()
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.split("(")[0].replace("void ", "")[:60]
        agg[name][0] += 1
        agg[name][1] += e.device_time
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'calls/it':>8s} {'mean us':>9s} {'us/it':>9s}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:60s} {c / iters:8.1f} {t / c:9.2f} {t / iters:9.2f}")
print(f"{'total':60s} {'':8s} {'':9s} {tot / iters:9.2f}")
