for D in "-DNIRC_TRACE_MINB_BVH=10" "-DNIRC_TRACE_MINB_BVH=12"; do
echo "== $D"
NIRC_NVCC_DEFS="$D" python -c "from paper_2412_04634_b200 import build; build.build(force=True)" > /dev/null || exit 1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --frame-steps 10 --no-extra-frames | python -c "
import json,sys; d=json.load(sys.stdin); f=d['frame_1080p']; q=f['sequential']
print(round(f['value'],3), {k:round(q[k],3) for k in ('value','render_collect_ms')})"
timeout 300 python tools/bvh_bench.py 2>&1 | grep '"pt"'
done
