"""Median per-stage device times (trace / inference / accumulate) of the
sequential cfg3 frame (bench.frame_bench with the C-ABI stage timer)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

w, h = (int(x) for x in os.environ.get("RES", "1920x1080").split("x"))
r = bench.frame_bench(int(sys.argv[1]) if len(sys.argv) > 1 else 6, 2, w, h)
print("STAGES " + json.dumps({"frame_ms": r["value"], **r["stage_ms"]}))
