mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv \
  --log-file gpurun_out/launches_cfg2_final.csv python bench.py --steps 3 --warmup 1 --no-frame --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_frame_final.csv python tools/profile_frame.py 3 > /dev/null 2>&1
cat gpurun_out/bench_full.json | head -c 3000
