import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2412_04634_b200 import _lib
from paper_2412_04634_b200.caches import Cache
from paper_2412_04634_b200.estimators import render_device
from paper_2412_04634_b200.frame import config3
from paper_2412_04634_b200.scene import load_builtin
os.environ["NIRC_INFER_ABLATE"] = "7"
lib = _lib.load()
buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
sc = load_builtin("cornell").with_resolution(64, 64)
cache = Cache.create("nirc", sc, seed=0, init="random")
lib.nirc_debug_infer_probe(C.c_void_p(buf.data_ptr()))
try:
    render_device(sc, config3(), cache)
    torch.cuda.synchronize()
except Exception as e:
    print("render raised", e)
f = buf.cpu().numpy().view(np.float32)
D = f[:128 * 32].reshape(128, 32)
img = f[4096:4096 + 64]
bias = f[4200:4264]
print("bias layer1[:8]", bias[:8])
print("image[:16]", img[:16])
print("D lane0[:8]", D[0, :8], "lane77[:8]", D[77, :8])
print("D == bias everywhere:", np.array_equal(D, np.tile(bias[:32], (128, 1))))
