mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for ND in 0 4 5; do
NIRC_DENSE_LEVELS=$ND timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-frame | python -c "import json,sys; d=json.load(sys.stdin); print('cfg2 dense levels $ND', d['value']/1e9, 'Gq/s', d['roofline']['avg_launch_ms'], 'ms')"
done
timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --frame-steps 10 | python -c "import json,sys; d=json.load(sys.stdin)['frame_1080p']; print({k:d[k] for k in ('value','render_collect_ms','record_allgather_ms','train_ms')})"
