"""Per-step latency of the fused training step for small batches (the
per-rank share of a sharded step, cfg1): B records -> B/128 API tiles."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2412_04634_b200.caches import train_frame_device  # noqa: E402
from paper_2412_04634_b200.mlp import init_theta, make_spec  # noqa: E402
from paper_2412_04634_b200.adam import AdamState  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
import nirc_oracle as O  # noqa: E402

from paper_2412_04634_b200.caches import Records  # noqa: E402

spec = make_spec(depth=4)
for B in (1024, 2048, 4096, 8192, 16384):
    r = O.synth_records(B, seed=3)
    rec = Records(kind="nirc", frame=0, n=B, **{k: torch.as_tensor(v).cuda() for k, v in r.items()})
    theta = torch.from_numpy(init_theta(spec, seed=1, out_scale=0.1)).cuda()
    adam = AdamState(theta)
    for _ in range(3):
        train_frame_device(spec, theta, rec, seed=0, frame=0, steps=4, adam=adam)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        train_frame_device(spec, theta, rec, seed=0, frame=0, steps=4, adam=adam)
    e1.record()
    torch.cuda.synchronize()
    print(B, "ms per 4-step frame", round(e0.elapsed_time(e1) / 10, 3))
