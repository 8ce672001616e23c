mkdir -p gpurun_out
for MB in 4 3; do
  NIRC_TRACE_MINB=$MB python -c "from paper_2412_04634_b200 import build; build.build(force=True)" || exit 1
  [ $MB = 4 ] && timeout 900 python -m pytest tests/test_gpu_render.py -x -q 2>&1 | tail -2
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --frame-steps 10 --no-extra-frames > gpurun_out/bench_mb$MB.json
  python -c "
import json; d=json.load(open('gpurun_out/bench_mb$MB.json')); f=d['frame_1080p']
print('MINB $MB', {k:round(f[k],3) for k in ('value','render_collect_ms','train_ms')})"
done
