"""Pinned / pageable host<->device copy bandwidth on this box (context for
the e2e number, which is PCIe-bound)."""
import json
import subprocess

import torch

n = 256 << 20
res = {}
for pinned in (True, False):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=pinned)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[f"{name}_{'pinned' if pinned else 'pageable'}_GBs"] = round(
            10 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
try:
    res["pcie"] = subprocess.run(
        ["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,"
         "pcie.link.gen.max", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    res["numa"] = subprocess.run(["bash", "-c", "nvidia-smi topo -m | head -3"],
                                 capture_output=True, text=True).stdout.strip()
except Exception as e:  # noqa: BLE001
    res["err"] = str(e)
print(json.dumps(res))
