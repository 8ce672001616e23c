timeout 300 python tools/infer_ab.py 0 2 2>&1 | grep -E "image|AB" | cut -c1-100
timeout 300 python tools/infer_timeline.py 2>&1 | tail -9
