mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_frame2.csv python tools/profile_frame.py 3 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_trace|k_infer_tc|k_train_tile' -s 6 -c 3 \
  -o gpurun_out/frame2 python tools/profile_frame.py 2 > gpurun_out/ncu_frame2.log 2>&1
ls gpurun_out
