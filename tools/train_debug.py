"""Stage-by-stage dump of k_train_tc (nirc_debug_train_probe) against the
oracle on one small batch: X, hidden pre-activations, output, dX."""
import ctypes as C
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import nirc_oracle as O  # noqa: E402
from paper_2412_04634_b200 import _lib  # noqa: E402
from paper_2412_04634_b200.caches import Records, train_frame_device  # noqa: E402
from paper_2412_04634_b200.mlp import init_theta, make_spec  # noqa: E402

depth = int(os.environ.get("DEPTH", 4))
n = int(os.environ.get("N_REC", 3000))
spec = make_spec(depth=depth, table=2 ** 12)
os_ = O.Spec(table=2 ** 12, depth=depth)
rec = O.synth_records(n, seed=5)
th = init_theta(spec, seed=3, out_scale=float(os.environ.get("OUT_SCALE", 0.05)))
B = min(n, 16384)
S = 336
dbg = torch.zeros((B, S), dtype=torch.float32, device="cuda")
lib = _lib.load()
lib.nirc_debug_train_probe.argtypes = [C.c_void_p]
lib.nirc_debug_train_probe(C.c_void_p(dbg.data_ptr()))
theta = torch.from_numpy(th.copy()).cuda()
res = train_frame_device(spec, theta, Records(kind="nirc", frame=2, **rec), seed=7, frame=2,
                         steps=1, return_idx=True)
lib.nirc_debug_train_probe(C.c_void_p(0))
d = dbg.cpu().numpy()
sel = res.batch_idx[0]
X, ent, wts = O.encode_batch(os_, th, rec["pos"][sel], rec["ns"][sel], rec["alb"][sel],
                             rec["rough"][sel], rec["dirs"][sel])
y, (acts, zs) = O.mlp_forward(os_, th, X, training=True)
_, dy = O.loss_relative_l2(y, rec["target"][sel], rec["pdf"][sel])
dy = dy.astype(np.float32)
dz = dy * (zs[-1] >= 0)
for l in range(os_.nl - 1, -1, -1):
    da = dz @ os_.W(th, l)
    if l > 0:
        dz = da * (zs[l - 1] >= 0)
dX = da


def cmp(name, a, b):
    err = np.abs(a - b)
    sc = np.abs(b).max() + 1e-30
    i = np.unravel_index(np.argmax(err), err.shape)
    print(f"{name:8s} max|ref| {sc:.3e} max err {err.max():.3e} (rel {err.max() / sc:.2e}) at {i}: "
          f"got {a[i]:.6e} want {b[i]:.6e}")


print("unsafe rows:", int((d[:, 308:310] > 0).any(axis=1).sum()), "of", B)
cmp("X", d[:, :47], X)
for l in range(os_.nl - 1):
    cmp(f"Z{l}", d[:, 48 + 64 * l: 48 + 64 * l + 64], zs[l])
cmp("out", d[:, 304:307], zs[-1])
cmp("dX", d[:, 312:336], dX[:, :24])
print("loss", res.trace)

# raw gradient (nirc_train_grad, before Adam) per parameter block
from paper_2412_04634_b200 import _dev  # noqa: E402

recs = Records(kind="nirc", frame=2, **rec)
r_c, _keep = recs.c_struct()
cs = _lib.make_c_spec(spec)
ntiles = lib.nirc_train_tiles(n, 16384)
grad = torch.zeros(spec.theta_len, dtype=torch.float32, device="cuda")
aux = torch.zeros(2, dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
need = lib.nirc_train_workspace_bytes(cs, n, 16384)
ws = torch.empty(need, dtype=torch.uint8, device="cuda")
_lib.check(lib.nirc_train_grad(cs, _dev.ptr(theta0 := torch.from_numpy(th.copy()).cuda()), r_c, 7,
                               2, 0, 16384, 1, 0.01, None, 0, ntiles, _dev.ptr(grad), _dev.ptr(aux),
                               _dev.ptr(flags), None, _dev.ptr(ws), int(ws.numel()),
                               _dev.stream()), "nirc_train_grad")
got = grad.cpu().numpy().astype(np.float64)
want = O.mlp_backward(os_, th, (acts, zs), dy, ent, wts).astype(np.float64)
for l in range(os_.nl):
    w0, b0 = int(spec.w_off[l]), int(spec.b_off[l])
    nw = int(spec.dims[l]) * int(spec.dims[l + 1])
    for nm, lo, hi in (("W", w0, w0 + nw), ("b", b0, b0 + int(spec.dims[l + 1]))):
        a, b = got[lo:hi], want[lo:hi]
        print(f"layer {l} {nm}: rel {np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30):.3e} "
              f"|want| {np.linalg.norm(b):.3e} |got| {np.linalg.norm(a):.3e}")
a, b = got[: spec.grid_len], want[: spec.grid_len]
print(f"grid: rel {np.linalg.norm(a - b) / np.linalg.norm(b):.3e}")

# two optimizer steps: device train_frame vs the oracle's train_step x 2
thA = torch.from_numpy(th.copy()).cuda()
resA = train_frame_device(spec, thA, Records(kind="nirc", frame=2, **rec), seed=7, frame=2,
                          steps=2)
thO = th.copy()
adamO = O.Adam(thO.size)
vals = []
for s in range(2):
    v, _ = O.train_step(os_, thO, adamO, rec, seed=7, frame=2, step=s)
    vals.append(v)
print("2-step loss device", resA.trace, "oracle", vals)
dth = thA.cpu().numpy() - thO
print("theta diff max", np.abs(dth).max(), "frac moved >1e-5", (np.abs(dth) > 1e-5).mean())
for l in range(os_.nl):
    w0 = int(spec.w_off[l])
    nw = int(spec.dims[l]) * int(spec.dims[l + 1])
    print(f"layer {l} W theta diff max {np.abs(dth[w0:w0 + nw]).max():.3e}")
