#!/bin/bash
# ncu --set full captures of the main training DFP kernels (one launch each), for profiles/.
mkdir -p gpurun_out
for k in rowreduce_kernel bnback_apply_kernel maxpool_argmax_kernel pool_back_kernel mask_kernel chain_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 6 -c 1 \
    -o gpurun_out/train_$k -f python scripts/profile_steps.py train > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
