mkdir -p gpurun_out
for M in 5 6; do
echo "== MINB $M"
NIRC_TRACE_MINB=$M python -c "from paper_2412_04634_b200 import build; build.build(force=True)" > /dev/null || exit 1
timeout 600 python tools/bvh_bench.py 2>&1 | grep scene_prims | grep '"pt"'
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --frame-steps 10 --no-extra-frames | python -c "
import json,sys; d=json.load(sys.stdin); f=d['frame_1080p']
print({k:round(f[k],3) for k in ('value','render_collect_ms','train_ms')})"
done
