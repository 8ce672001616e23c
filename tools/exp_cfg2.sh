mkdir -p gpurun_out
for DEFS in "" "-DNIRC_FF_NOSTREAM" "-DNIRC_FF_F64SH" "-DNIRC_FF_NOSTREAM -DNIRC_FF_F64SH"; do
  NIRC_NVCC_DEFS="$DEFS" python -c "from paper_2412_04634_b200 import build; build.build(force=True)" || exit 1
  for rep in 1 2; do
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-frame | python -c "import json,sys; d=json.load(sys.stdin); print('cfg2 [$DEFS]', round(d['value']/1e9,3), 'Gq/s', round(d['roofline']['avg_launch_ms'],4), 'ms')"
  done
done
python -c "from paper_2412_04634_b200 import build; build.build(force=True)"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_full_forward_tc -s 2 -c 1 \
  -o gpurun_out/full_forward_r1b python bench.py --steps 3 --warmup 1 --no-frame --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
