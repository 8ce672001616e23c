mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
for rep in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --frame-steps 10 --no-extra-frames | python -c "
import json,sys; d=json.load(sys.stdin); f=d['frame_1080p']; q=f['sequential']
print(round(d['value']/1e9,3), round(f['value'],3), {k:round(q[k],3) for k in ('value','render_collect_ms','train_ms')})"
done
