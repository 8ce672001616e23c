"""One 4-step training frame at B=2048 (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
import torch  # noqa: E402
import nirc_oracle as O  # noqa: E402

from paper_2412_04634_b200.adam import AdamState  # noqa: E402
from paper_2412_04634_b200.caches import Records, train_frame_device  # noqa: E402
from paper_2412_04634_b200.mlp import init_theta, make_spec  # noqa: E402

spec = make_spec(depth=4)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
r = O.synth_records(B, seed=3)
rec = Records(kind="nirc", frame=0, n=B, **{k: torch.as_tensor(v).cuda() for k, v in r.items()})
theta = torch.from_numpy(init_theta(spec, seed=1, out_scale=0.1)).cuda()
adam = AdamState(theta)
for _ in range(3):
    train_frame_device(spec, theta, rec, seed=0, frame=0, steps=4, adam=adam)
torch.cuda.synchronize()
