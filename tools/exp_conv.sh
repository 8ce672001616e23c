mkdir -p gpurun_out
for S in 2 4; do
NIRC_NVCC_DEFS="-DNIRC_TRAIN_SPLIT=$S" python -c "from paper_2412_04634_b200 import build; build.build(force=True)" > /dev/null || exit 1
for rep in 1 2; do echo "== split $S rep $rep"; timeout 300 python tools/exp_conv.py gpurun_out/conv_${S}_${rep}.npy; done
done
