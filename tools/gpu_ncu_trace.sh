mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_trace|k_infer_tc' -s 2 -c 2 \
  -o gpurun_out/frame4 python tools/profile_frame.py 2 > gpurun_out/ncu_frame4.log 2>&1
ls gpurun_out | grep frame4
