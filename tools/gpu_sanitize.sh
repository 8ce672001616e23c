#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the small
# launches of tools/sanitize_run.py; logs into gpurun_out/sanitize_*.log
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --target-processes all \
    python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
