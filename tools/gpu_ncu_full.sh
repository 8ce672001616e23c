#!/bin/bash
# ncu --set full captures of the dominant kernels (one launch each).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_full_forward_tc -s 2 -c 1 \
  -o gpurun_out/full_forward python bench.py --steps 3 --warmup 1 --no-frame --no-cpu-baseline > gpurun_out/ncu_full_ff.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_trace|k_infer_tc|k_walk_record|k_train_tile|k_reduce_grad' -s 10 -c 5 \
  -o gpurun_out/frame python tools/profile_frame.py 2 > gpurun_out/ncu_full_frame.log 2>&1
ls -la gpurun_out
