mkdir -p gpurun_out
for F in 0 1; do
  NIRC_RENDER_FMAD=$F python -c "from paper_2412_04634_b200 import build; build.build(force=True)"
  timeout 600 python -m pytest tests/test_gpu_render.py -x -q 2>&1 | tail -3
  timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --frame-steps 10 | python -c "import json,sys; d=json.load(sys.stdin)['frame_1080p']; print('FMAD',$F,{k:d[k] for k in ('value','render_ms','collect_ms','train_ms')})"
done
