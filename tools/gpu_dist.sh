#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_dist.log 2>&1
tail -3 gpurun_out/pytest_dist.log
NIRC_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --frame-steps 3 \
  > gpurun_out/bench2.json 2> gpurun_out/bench2.err
tail -5 gpurun_out/bench2.err
cat gpurun_out/bench2.json
