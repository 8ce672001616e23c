#!/bin/bash
# One GPU round trip: gpu tests, smoke, default bench, ncu launch lists.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 1 --no-frame --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_frame.csv python tools/profile_frame.py 3 > gpurun_out/ncu_frame.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/bench.json
