mkdir -p gpurun_out
for U in 1 2 4 8; do
  NIRC_NVCC_DEFS="-DNIRC_FILTER_UNROLL=$U" python -c "from paper_2412_04634_b200 import build; build.build(force=True)" || exit 1
  timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --frame-steps 10 --no-extra-frames > gpurun_out/b.json
  python -c "
import json; d=json.load(open('gpurun_out/b.json')); f=d['frame_1080p']
print('UNROLL $U', {k:round(f[k],3) for k in ('value','render_collect_ms','train_ms')})"
done
python -c "from paper_2412_04634_b200 import build; build.build(force=True)"
