mkdir -p gpurun_out
RES=3840x2160 NC=16,16 timeout 600 python tools/infer_ab.py 0 2 2>&1 | grep -E "image|AB" | cut -c1-120 | sed 's/^/4k /'
RES=128x128 NC=8 timeout 300 python tools/infer_ab.py 0 2 2>&1 | grep -E "image|AB" | cut -c1-120 | sed 's/^/128 /'
timeout 900 python -m pytest tests/test_gpu_render.py tests/test_gpu_frame_pipeline.py tests/test_gpu_trained.py -x -q 2>&1 | tail -3
