# same-box cfg2 A/B over in-tree builds libnirc_b200_<name>.so (device q/s of
# bench.py's cfg2 leg, three repetitions)
for rep in 1 2 3; do
  for v in "$@"; do
    NIRC_LIB_PATH=$PWD/paper_2412_04634_b200/libnirc_b200_$v.so timeout 300 python bench.py --steps 50 --warmup 5 --no-frame --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['roofline']['avg_launch_ms'])"
  done
done
