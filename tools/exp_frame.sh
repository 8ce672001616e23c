mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_render.py tests/test_gpu_api.py tests/test_gpu_edges.py -q -x 2>&1 | tail -2
for rep in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --frame-steps 10 | python -c "
import json,sys; d=json.load(sys.stdin); f=d['frame_1080p']
print('cfg2', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), {k:round(f[k],3) for k in ('value','render_collect_ms','train_ms')}, '4k', round(f['cfg5_4k']['value'],2), '128', round(f['cfg1_128']['value'],3))"
done
