# same-box A/B over several in-tree builds: libnirc_b200_<name>.so for each
# name given (stage times of the sequential 1080p frame, two repetitions)
for rep in 1 2; do
  for v in "$@"; do
    NIRC_LIB_PATH=$PWD/paper_2412_04634_b200/libnirc_b200_$v.so timeout 300 python tools/stage_times.py 8 2>&1 | grep STAGES | sed "s/^/$v /"
  done
done
