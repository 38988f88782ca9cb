#!/bin/bash
# One GPU session: parity tests, bench (both arms), launch list, DRAM traffic per conv launch, and
# one full ncu capture of the fused conv kernel. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 120 python scripts/profile_steps.py infer fuse > gpurun_out/steps_infer.txt 2>&1
timeout 300 python scripts/profile_steps.py train > gpurun_out/steps_train.txt 2>&1
SOL_BENCH_NO_LAUNCH_COUNT=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-train --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?"
SOL_BENCH_NO_LAUNCH_COUNT=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"igemm_ws_kernel|stem_kernel|stem_row_kernel|halo_kernel" -c 60 --csv --log-file gpurun_out/conv_traffic.csv \
  python bench.py --steps 1 --warmup 1 --no-train --no-cpu-baseline > gpurun_out/ncu_traffic.log 2>&1; echo "ncu2 rc=$?"
SOL_BENCH_NO_LAUNCH_COUNT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:igemm_ws_kernel --launch-skip 20 -c 1 \
  -o gpurun_out/conv_fused_full -f python bench.py --steps 1 --warmup 1 --no-train --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu3 rc=$?"
