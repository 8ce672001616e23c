# A/B of two in-tree builds of the library: the default one and libnirc_b200_base.so
for rep in 1 2; do
  for v in base new; do
    if [ $v = base ]; then export NIRC_LIB_PATH=$PWD/paper_2412_04634_b200/libnirc_b200_base.so; else unset NIRC_LIB_PATH; fi
    timeout 300 python tools/stage_times.py 8 2>&1 | grep STAGES | sed "s/^/$v /"
  done
done
