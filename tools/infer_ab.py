"""A/B of the frame inference kernels on the cfg3 (or RES=WxH, NC=16[,16])
two-level frame: render time with CUDA events (median of 10 after 3
warm-ups) for each NIRC_INFER_NP setting given on the command line (0 = the
grouped k_infer_tc, 1/2/4 = k_infer_ws with that many producer warpgroups),
each in its own process; image agreement against the first setting; and
the k_infer_ws phase stamps of CTA 0 (chain group 0 / producer 0).

    python tools/infer_ab.py 0 2 1
"""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import numpy as np
    import torch

    from paper_2412_04634_b200 import _lib
    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.estimators import render_device
    from paper_2412_04634_b200.frame import config3
    from paper_2412_04634_b200.scene import load_builtin

    w, h = (int(x) for x in os.environ.get("RES", "1920x1080").split("x"))
    nc = tuple(int(x) for x in os.environ.get("NC", "16").split(","))
    sc = load_builtin("cornell").with_resolution(w, h)
    cache = Cache.create("nirc", sc, seed=0, init="random")
    cfg = config3(nc)
    for _ in range(3):
        render_device(sc, cfg, cache)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        img, img2, term, q = render_device(sc, cfg, cache)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out = {"np": os.environ.get("NIRC_INFER_NP"), "render_ms": sorted(ts)[len(ts) // 2],
           "queries": int(q.item())}
    np.save(os.environ["AB_OUT"], img.cpu().numpy() if hasattr(img, "cpu") else np.asarray(img))
    lib = _lib.load()
    buf = torch.zeros(4096, dtype=torch.int64, device="cuda")
    lib.nirc_debug_infer_probe(C.c_void_p(buf.data_ptr()))
    render_device(sc, cfg, cache)
    torch.cuda.synchronize()
    lib.nirc_debug_infer_probe(None)
    a = buf.cpu().numpy().astype(np.float64)
    if os.environ.get("NIRC_INFER_NP", "2") != "0":
        ch = a[:32 * 16].reshape(32, 16)
        pr = a[2048:2048 + 32 * 8].reshape(32, 8)
        ok = ch[:, 0] > 0
        if ok.sum() > 6:
            c = ch[ok][2:]
            out["chain_tile_cycles"] = float(np.median(np.diff(c[:, 0])))
            out["chain_wait_full"] = float(np.median(c[:, 1] - c[:, 0]))
            out["chain_layers"] = [float(np.median(c[:, 3 + l] - c[:, 2 + l])) for l in range(4)]
            out["chain_combine"] = float(np.median(c[:, 8] - c[:, 6]))
            # layer 1 detail: ld/split/st, prefill+wait, barrier, issue, MMA (issue->done)
            out["layer1_split"] = float(np.median(c[:, 9] - c[:, 3]))
            out["layer1_prefill"] = float(np.median(c[:, 10] - c[:, 9]))
            out["layer1_bar"] = float(np.median(c[:, 11] - c[:, 10]))
            out["layer1_issue"] = float(np.median(c[:, 12] - c[:, 11]))
            out["layer2_mma_wait"] = float(np.median(c[:, 4] - c[:, 12]))
        okp = pr[:, 0] > 0
        if okp.sum() > 6:
            p = pr[okp][2:]
            out["prod_tile_cycles"] = float(np.median(np.diff(p[:, 0])))
            out["prod_phases"] = [float(np.median(p[:, k + 1] - p[:, k])) for k in range(4)]
    print("AB " + json.dumps(out), flush=True)


def main():
    if os.environ.get("AB_CHILD"):
        child()
        return
    import numpy as np

    settings = sys.argv[1:] or ["0", "2"]
    imgs = []
    for s in settings:
        out = f"/tmp/ab_{s}.npy"
        env = dict(os.environ, AB_CHILD="1", NIRC_INFER_NP=s, AB_OUT=out)
        try:
            r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True,
                               timeout=240)
        except subprocess.TimeoutExpired:
            print(f"setting {s}: TIMEOUT", flush=True)
            continue
        line = [l for l in r.stdout.splitlines() if l.startswith("AB ")]
        print(line[0] if line else r.stdout[-2000:] + r.stderr[-3000:], flush=True)
        if os.path.exists(out):
            imgs.append((s, np.load(out)))
    if len(imgs) > 1:
        s0, i0 = imgs[0]
        for s, im in imgs[1:]:
            d = np.abs(im - i0)
            rel = d / np.maximum(np.abs(i0), 1e-3)
            print(f"image {s} vs {s0}: max abs {d.max():.3e}  max rel {rel.max():.3e}  "
                  f"mean rel {rel.mean():.3e}  finite {np.isfinite(im).all()}")


if __name__ == "__main__":
    main()
