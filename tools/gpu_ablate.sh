mkdir -p gpurun_out
for ab in 0 1 2; do
  NIRC_INFER_ABLATE=$ab timeout 300 python tools/infer_ab.py 2 2>&1 | grep AB | sed "s/^/ablate=$ab /" | cut -c1-140
done
