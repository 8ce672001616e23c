# round-end evidence: frame launch list + full captures of the frame's kernels and cfg2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_frame_r1f.csv python tools/profile_frame.py 3 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_trace|k_infer_tc|k_train_tile' -s 6 -c 3 \
  -o gpurun_out/frame_r1f python tools/profile_frame.py 2 > gpurun_out/ncu_frame_r1f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'k_full_forward_tc' -s 2 -c 1 \
  -o gpurun_out/cfg2_r1f python bench.py --steps 3 --warmup 1 --no-frame --no-cpu-baseline > gpurun_out/ncu_cfg2_r1f.log 2>&1
ls gpurun_out
