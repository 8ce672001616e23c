mkdir -p gpurun_out
for S in 4 2; do
echo "== split $S"
NIRC_NVCC_DEFS="-DNIRC_TRAIN_SPLIT=$S" python -c "from paper_2412_04634_b200 import build; build.build(force=True)" > /dev/null || exit 1
timeout 900 python -m pytest tests -q -x -m gpu -k "train or distributed or converg or snapshot" 2>&1 | tail -2
for rep in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --frame-steps 10 --no-extra-frames | python -c "
import json,sys; d=json.load(sys.stdin); f=d['frame_1080p']
print({k:round(f[k],3) for k in ('value','render_collect_ms','train_ms')})"
done
done
