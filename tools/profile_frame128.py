"""A few cfg1 frames (128^2 Cornell, two-level nc=(8,)) for ncu / nsys-less timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
print(bench.frame_bench(frames, 1, 128, 128, (8,), name="cfg1"))
