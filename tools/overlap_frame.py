"""Overlapped cfg3 frame time (bench.frame_bench_overlap) -- for scheduling
experiments (e.g. NIRC_TRACE_PER_SM)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.frame_bench_overlap(int(sys.argv[1]) if len(sys.argv) > 1 else 8, 3)
print("OVERLAP " + json.dumps({"frame_ms": r["value"], "train_span_ms": r.get("train_stream_span_ms")}))
