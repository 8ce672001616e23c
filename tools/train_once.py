"""One cfg3-sized 4-step train_frame (113,895 records, D = 4) after one
warm-up frame -- the command profiled by ncu for the training launch list."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
import torch  # noqa: E402

import nirc_oracle as O  # noqa: E402
from paper_2412_04634_b200.adam import AdamState  # noqa: E402
from paper_2412_04634_b200.caches import Records, train_frame_device  # noqa: E402
from paper_2412_04634_b200.mlp import init_theta, make_spec  # noqa: E402

n = int(os.environ.get("N_REC", 113895))
spec = make_spec(depth=4)
r = O.synth_records(n, seed=3)
rec = Records(kind="nirc", frame=0, n=n, **{k: torch.as_tensor(v).cuda() for k, v in r.items()})
theta = torch.from_numpy(init_theta(spec, seed=1, out_scale=0.1)).cuda()
adam = AdamState(theta)
for _ in range(2):
    train_frame_device(spec, theta, rec, seed=0, frame=0, steps=4, adam=adam)
torch.cuda.synchronize()
