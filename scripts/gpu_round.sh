#!/bin/bash
# One GPU session of evidence for profiles/: per-step times (inference + training), launch lists
# (ncu gpu__time_duration + DRAM bytes per launch) of one inference and one training step, the
# DRAM traffic of every conv launch, and one full ncu capture each of the dominant inference conv
# kernel and the training weight-gradient kernel. Outputs under gpurun_out/ (copy summaries to
# profiles/ with scripts/summarize_launches.py / scripts/summarize_ncu.py).
mkdir -p gpurun_out
timeout 300 python scripts/profile_steps.py infer fuse > gpurun_out/steps_infer.txt 2>&1
timeout 300 python scripts/profile_steps.py train > gpurun_out/steps_train.txt 2>&1
export SOL_BENCH_NO_LAUNCH_COUNT=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/launches_infer.csv \
  python bench.py --steps 2 --warmup 1 --no-train --no-cpu-baseline --no-configs > gpurun_out/ncu_li.log 2>&1; echo "ncu infer rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 900 --csv --log-file gpurun_out/launches_train.csv \
  python scripts/diag/one_train_step.py > gpurun_out/ncu_lt.log 2>&1; echo "ncu train rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:igemm_ws_kernel --launch-skip 20 -c 1 \
  -o gpurun_out/r02_conv_full -f python bench.py --steps 1 --warmup 1 --no-train --no-cpu-baseline --no-configs > gpurun_out/ncu_cf.log 2>&1; echo "ncu conv rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wgrad_halo_kernel -c 1 \
  -o gpurun_out/r02_wgrad_full -f python scripts/wgrad_micro.py l1.conv2 --ncu > gpurun_out/ncu_wf.log 2>&1; echo "ncu wgrad rc=$?"
