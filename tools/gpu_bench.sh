mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 3000 gpurun_out/bench.json; echo; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench.err
