"""Phase timestamps (clock64, CTA 0 / thread 0) of k_train_tc on the
cfg3-sized training batch (nirc_debug_train_phases)."""
import ctypes as C
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
import torch  # noqa: E402

import nirc_oracle as O  # noqa: E402
from paper_2412_04634_b200 import _lib  # noqa: E402
from paper_2412_04634_b200.adam import AdamState  # noqa: E402
from paper_2412_04634_b200.caches import Records, train_frame_device  # noqa: E402
from paper_2412_04634_b200.mlp import init_theta, make_spec  # noqa: E402

n = 113895
spec = make_spec(depth=4)
r = O.synth_records(n, seed=3)
rec = Records(kind="nirc", frame=0, n=n, **{k: torch.as_tensor(v).cuda() for k, v in r.items()})
theta = torch.from_numpy(init_theta(spec, seed=1, out_scale=0.1)).cuda()
adam = AdamState(theta)
lib = _lib.load()
buf = torch.zeros(80, dtype=torch.int64, device="cuda")
lib.nirc_debug_train_phases.argtypes = [C.c_void_p]
for _ in range(3):
    train_frame_device(spec, theta, rec, seed=0, frame=0, steps=4, adam=adam)
lib.nirc_debug_train_phases(C.c_void_p(buf.data_ptr()))
train_frame_device(spec, theta, rec, seed=0, frame=0, steps=1, adam=adam)
lib.nirc_debug_train_phases(C.c_void_p(0))
t = buf.cpu().numpy()
names = {0: "prologue", 1: "encode", 2: "weights+issue0", 3: "fwd L0", 4: "fwd L1", 5: "fwd L2",
         6: "fwd L3", 8: "fwd out", 9: "loss"}
for l in range(4, -1, -1):
    names[10 + 5 * l] = f"bwd{l} maxima"
    names[11 + 5 * l] = f"bwd{l} operands"
    names[12 + 5 * l] = f"bwd{l} mma"
    names[13 + 5 * l] = f"bwd{l} epilogue"
names[40] = "bwd0 partial stores"
names[41] = "scatter"
names[42] = "barrier"
names[43] = "flush"
order = [k for k in [0, 1, 2, 3, 4, 5, 6, 8, 9] + [x for l in range(4, -1, -1) for x in
         (10 + 5 * l, 11 + 5 * l, 12 + 5 * l, 13 + 5 * l)] + [40, 41, 42, 43] if t[k] != 0]
prev = t[order[0]]
print("cycles since the previous mark (1.9 GHz: 1 us = 1900 cycles)")
for k in order:
    print(f"{names.get(k, k):22s} {t[k] - prev:8d}")
    prev = t[k]
print("total", t[order[-1]] - t[order[0]])
for base, who in ((48, "thread 0 (h = 0)"), (56, "thread 128 (h = 1)")):
    e = t[base: base + 6]
    print(who, "idx", e[1] - e[0], "u", e[2] - e[1], "static", e[3] - e[2], "tma wait", e[4] - e[3],
          "levels", e[5] - max(e[4], e[2]))
