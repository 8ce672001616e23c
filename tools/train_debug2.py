"""Step-2 localisation: theta after one device step vs the oracle, then the
stage dump + raw gradient of the SECOND step's batch at the device theta."""
import ctypes as C
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import nirc_oracle as O  # noqa: E402
from paper_2412_04634_b200 import _dev, _lib  # noqa: E402
from paper_2412_04634_b200.caches import Records, train_frame_device  # noqa: E402
from paper_2412_04634_b200.mlp import init_theta, make_spec  # noqa: E402

n = 3000
spec = make_spec(depth=4, table=2 ** 12)
os_ = O.Spec(table=2 ** 12, depth=4)
rec = O.synth_records(n, seed=5)
th = init_theta(spec, seed=3)
lib = _lib.load()
thD = torch.from_numpy(th.copy()).cuda()
train_frame_device(spec, thD, Records(kind="nirc", frame=2, **rec), seed=7, frame=2, steps=1)
th1 = th.copy()
O.train_step(os_, th1, O.Adam(th1.size), rec, seed=7, frame=2, step=0)
d = thD.cpu().numpy() - th1
print("theta after 1 step: max diff", np.abs(d).max(), "n>1e-5", int((np.abs(d) > 1e-5).sum()))
for l in range(os_.nl):
    w0 = int(spec.w_off[l]); nw = int(spec.dims[l]) * int(spec.dims[l + 1])
    b0 = int(spec.b_off[l])
    print(f" layer {l}: W {np.abs(d[w0:w0+nw]).max():.3e}  b {np.abs(d[b0:b0+int(spec.dims[l+1])]).max():.3e}")
print(" grid", np.abs(d[:spec.grid_len]).max())
# second step's raw gradient at the device theta
thd = thD.cpu().numpy()
sel = O.select_batch(7, 2, 1, n)
X, ent, wts = O.encode_batch(os_, thd, rec["pos"][sel], rec["ns"][sel], rec["alb"][sel],
                             rec["rough"][sel], rec["dirs"][sel])
y, cache = O.mlp_forward(os_, thd, X, training=True)
val, dy = O.loss_relative_l2(y, rec["target"][sel], rec["pdf"][sel])
want = O.mlp_backward(os_, thd, cache, dy.astype(np.float32), ent, wts).astype(np.float64)
recs = Records(kind="nirc", frame=2, **rec)
r_c, _keep = recs.c_struct()
cs = _lib.make_c_spec(spec)
grad = torch.zeros(spec.theta_len, dtype=torch.float32, device="cuda")
aux = torch.zeros(2, dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
ws = torch.empty(lib.nirc_train_workspace_bytes(cs, n, 16384), dtype=torch.uint8, device="cuda")
S = 336
dbg = torch.zeros((n, S), dtype=torch.float32, device="cuda")
lib.nirc_debug_train_probe.argtypes = [C.c_void_p]
lib.nirc_debug_train_probe(C.c_void_p(dbg.data_ptr()))
_lib.check(lib.nirc_train_grad(cs, _dev.ptr(thD), r_c, 7, 2, 1, 16384, 1, 0.01, None, 0,
                               lib.nirc_train_tiles(n, 16384), _dev.ptr(grad), _dev.ptr(aux),
                               _dev.ptr(flags), None, _dev.ptr(ws), int(ws.numel()),
                               _dev.stream()), "nirc_train_grad")
lib.nirc_debug_train_probe(C.c_void_p(0))
dd = dbg.cpu().numpy()
print("step2 loss dev", float(aux[0].item()) / (n * 3), "oracle", val,
      "unsafe rows", int((dd[:, 308:310] > 0).any(axis=1).sum()))
acts, zs = cache
for l in range(os_.nl - 1):
    e = np.abs(dd[:, 48 + 64 * l: 112 + 64 * l] - zs[l]).max()
    print(f" Z{l} max err {e:.3e}")
print(" out max err", np.abs(dd[:, 304:307] - zs[-1]).max(), "max|out|", np.abs(zs[-1]).max())
got = grad.cpu().numpy().astype(np.float64)
for l in range(os_.nl):
    w0, b0 = int(spec.w_off[l]), int(spec.b_off[l])
    nw = int(spec.dims[l]) * int(spec.dims[l + 1])
    for nm, lo, hi in (("W", w0, w0 + nw), ("b", b0, b0 + int(spec.dims[l + 1]))):
        a, b = got[lo:hi], want[lo:hi]
        print(f" layer {l} {nm}: rel {np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30):.3e}")
print(" grid rel", np.linalg.norm(got[:spec.grid_len] - want[:spec.grid_len]) / np.linalg.norm(want[:spec.grid_len]))
