for pv in 1 0; do
  NIRC_PAIRS=$pv timeout 300 python bench.py --steps 50 --warmup 5 --no-frame --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pairs=$pv', d['value'], d['roofline']['avg_launch_ms'])"
done
timeout 300 python tools/infer_ab.py 0 2 2>&1 | grep -E "image|AB" | cut -c1-90
timeout 600 python -m pytest tests/test_gpu_neural.py tests/test_gpu_api.py -x -q 2>&1 | tail -2
