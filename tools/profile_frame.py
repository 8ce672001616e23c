"""Runs a few cfg3 frames (1080p Cornell, two-level nc=(16,)) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
print(bench.frame_bench(frames, 1))
