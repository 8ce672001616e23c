timeout 300 python tools/infer_ab.py 0 2 2>&1 | grep -E "image|AB" | cut -c1-100
timeout 600 python -m pytest tests/test_gpu_render.py tests/test_gpu_trained.py tests/test_gpu_api.py -q 2>&1 | tail -2
