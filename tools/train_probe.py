"""Training-step probe: cfg3-sized record set (113,895 records -> 4 x 16,384
samples), D = 4 default spec.  Times the 4-step train_frame on the tcgen05
kernel and on the SIMT kernel (NIRC_TRAIN_SIMT=1), and compares the two
paths' losses / gradients (Adam m after one step = 0.1 g)."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import nirc_oracle as O  # noqa: E402
from paper_2412_04634_b200.adam import AdamState  # noqa: E402
from paper_2412_04634_b200.caches import Records, train_frame_device  # noqa: E402
from paper_2412_04634_b200.mlp import init_theta, make_spec  # noqa: E402

n = int(os.environ.get("N_REC", 113895))
spec = make_spec(depth=int(os.environ.get("DEPTH", 4)))
r = O.synth_records(n, seed=3)
rec = Records(kind="nirc", frame=0, n=n, **{k: torch.as_tensor(v).cuda() for k, v in r.items()})
th0 = init_theta(spec, seed=1, out_scale=0.1)


def run(simt, steps, reps, warm=3):
    if simt:
        os.environ["NIRC_TRAIN_SIMT"] = "1"
    else:
        os.environ.pop("NIRC_TRAIN_SIMT", None)
    theta = torch.from_numpy(th0.copy()).cuda()
    adam = AdamState(theta)
    res = train_frame_device(spec, theta, rec, seed=0, frame=0, steps=1, adam=adam)
    g = (adam.m / np.float32(0.1)).cpu().numpy().astype(np.float64)
    trace = res.trace
    for _ in range(warm):
        train_frame_device(spec, theta, rec, seed=0, frame=0, steps=steps, adam=adam)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        train_frame_device(spec, theta, rec, seed=0, frame=0, steps=steps, adam=adam)
    e1.record()
    torch.cuda.synchronize()
    return g, trace, e0.elapsed_time(e1) / reps


g_tc, tr_tc, t_tc = run(False, 4, 10)
g_si, tr_si, t_si = run(True, 4, 10)
print(f"4-step frame: tcgen05 {t_tc:.3f} ms   simt {t_si:.3f} ms   (n={n})")
print("loss step0", tr_tc, tr_si)
for name, lo, hi in (("mlp", spec.grid_len, spec.theta_len), ("grid", 0, spec.grid_len), ("all", 0, spec.theta_len)):
    a, b = g_tc[lo:hi], g_si[lo:hi]
    cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b) + 1e-300))
    rel = float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-300))
    print(f"grad {name}: cos {cos:.9f} rel {rel:.3e} |b| {np.linalg.norm(b):.3e}")
