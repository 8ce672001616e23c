mkdir -p gpurun_out
timeout 900 python tools/infer_ab.py ${AB_SETTINGS:-0 2 1 4} > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | cut -c1-160
if [ -n "$AB_TESTS" ]; then
  timeout 600 python -m pytest $AB_TESTS -x -q 2>&1 | tail -5
fi
