mkdir -p gpurun_out
for M in 0 1 32 100; do
  NIRC_NVCC_DEFS="-DNIRC_MBAR_MODE=$M" python -c "from paper_2412_04634_b200 import build; build.build(force=True)" || exit 1
  timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --frame-steps 10 --no-extra-frames > gpurun_out/b.json
  python -c "
import json; d=json.load(open('gpurun_out/b.json')); f=d['frame_1080p']
print('MBAR $M cfg2', round(d['value']/1e9,3), {k:round(f[k],3) for k in ('value','render_collect_ms','train_ms')})"
done
python -c "from paper_2412_04634_b200 import build; build.build(force=True)"
