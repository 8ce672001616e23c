# same-box A/B of the default build against libnirc_b200_base.so (stage
# times), the new build's k_infer_ws timeline, and the inference parity tests
bash tools/gpu_lib_ab.sh
NIRC_INFER_ABLATE=0 timeout 300 python tools/infer_timeline.py 2>&1 | tail -3
timeout 900 python -m pytest -q -x tests/test_gpu_trained.py tests/test_gpu_render.py 2>&1 | tail -3
