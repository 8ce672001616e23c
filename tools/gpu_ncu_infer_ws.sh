# one ncu --set full capture of k_infer_ws (cfg3 frame) with source
mkdir -p gpurun_out/ws
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_infer_ws -s 2 -c 1 \
  -o gpurun_out/ws/infer_ws -f python tools/profile_frame.py 2 > gpurun_out/ws/ncu.log 2>&1
tail -3 gpurun_out/ws/ncu.log
