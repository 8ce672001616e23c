mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_train.csv python tools/profile_frame.py 3 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_train_tile' -s 2 -c 1 \
  -o gpurun_out/train1 python tools/profile_frame.py 2 > gpurun_out/ncu_train1.log 2>&1
ls gpurun_out
