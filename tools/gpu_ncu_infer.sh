# one ncu --set full capture of the frame inference kernel (cfg3 frame)
mkdir -p gpurun_out
K=${NCU_KERNEL:-k_infer_ws}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 \
  -o gpurun_out/ncu_$K -f python tools/frame_once.py > gpurun_out/ncu_$K.log 2>&1
tail -3 gpurun_out/ncu_$K.log
