mkdir -p gpurun_out
for MB in 4 3; do
  NIRC_TRACE_MINB=$MB python -c "from paper_2412_04634_b200 import build; build.build(force=True)" || exit 1
  [ $MB = 4 ] && timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --frame-steps 10 > gpurun_out/bench_mb$MB.json
  python -c "
import json; d=json.load(open('gpurun_out/bench_mb$MB.json')); f=d['frame_1080p']
print('MINB $MB cfg2', d['value']/1e9, {k:f[k] for k in ('value','render_collect_ms','train_ms')})
print('  4k', {k:f['cfg5_4k'][k] for k in ('value','render_collect_ms','train_ms','queries_per_frame','records_per_frame')})
print('  128', {k:f['cfg1_128'][k] for k in ('value','render_collect_ms','train_ms')})"
done
