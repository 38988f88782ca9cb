#!/bin/bash
# Training conv kernels under ncu (time, DRAM bytes, tensor-pipe activity) for profiles/r02_train_conv.md:
# python scripts/summarize_train_conv.py gpurun_out/train_conv.csv
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:"wgrad|stem_kernel|igemm_ws_kernel|halo_kernel|interleave" -c 500 --csv \
  --log-file gpurun_out/train_conv.csv python scripts/profile_steps.py train > gpurun_out/ncu_tc.log 2>&1
echo "ncu rc=$?"
