#!/bin/bash
# Round-2 evidence from ONE build: GPU tests, smoke, default bench + the
# reference arm, ncu launch lists (cfg2 bench, cfg3 frame), ncu --set full of
# the dominant kernels, compute-sanitizer over the small launches.
mkdir -p gpurun_out/r2
O=gpurun_out/r2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_bench_cfg2.csv python bench.py --steps 3 --warmup 1 --no-frame --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches_frame_cfg3.csv python tools/profile_frame.py 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_full_forward_tc -s 2 -c 1 \
  -o $O/full_forward -f python bench.py --steps 3 --warmup 1 --no-frame --no-cpu-baseline > $O/ncu_ff.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_trace|k_infer_ws|k_train_tc|k_fixed_scatter' -s 8 -c 4 \
  -o $O/frame -f python tools/profile_frame.py 2 > $O/ncu_frame.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  extra=""; [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 50 \
    python tools/sanitize_run.py > $O/sanitize_$tool.log 2>&1
done
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
for t in memcheck racecheck synccheck initcheck; do grep -E "SUMMARY" $O/sanitize_$t.log; done
ls -la $O
