"""Per-call wall/device times of the e2e path (full_forward on pinned host f64
rows, 2^22 queries) to see how box-level PCIe variance shows up."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_04634_b200 import workloads  # noqa: E402
from paper_2412_04634_b200.mlp import full_forward, init_theta, make_spec  # noqa: E402

spec = make_spec(depth=2)
theta = torch.from_numpy(init_theta(spec, seed=1, out_scale=0.1)).cuda()
q = workloads.measure_queries_device(1 << 22, seed=0)
host = [torch.from_numpy(np.ascontiguousarray(a.cpu().numpy())).pin_memory() for a in q]
y = torch.empty((1 << 22, 3), dtype=torch.float32).pin_memory()
for _ in range(3):
    full_forward(spec, theta, *host, out=y)
torch.cuda.synchronize()
ts = []
for _ in range(40):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    full_forward(spec, theta, *host, out=y)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = np.array(ts)
print("ms per call: min %.2f median %.2f mean %.2f max %.2f" % (ts.min(), np.median(ts), ts.mean(), ts.max()))
print(np.round(ts, 2).tolist())
