# usage: bash tools/exp_defs.sh "<defs A>" "<defs B>" ...  (NIRC_NVCC_DEFS variants, frame timing)
mkdir -p gpurun_out
for D in "$@"; do
echo "== defs: $D"
NIRC_NVCC_DEFS="$D" python -c "from paper_2412_04634_b200 import build; build.build(force=True)" > /dev/null || exit 1
for rep in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --frame-steps 10 --no-extra-frames | python -c "
import json,sys; d=json.load(sys.stdin); f=d['frame_1080p']; q=f['sequential']
print(round(d['value']/1e9,3), round(f['value'],3), {k:round(q[k],3) for k in ('value','render_collect_ms','train_ms')})"
done
done
