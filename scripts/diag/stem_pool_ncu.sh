export SOL_BENCH_NO_LAUNCH_COUNT=1
SOL_STEM_POOL=1 timeout 300 python scripts/profile_steps.py infer fuse 2>&1 | grep -E "^total|conv_stem|dfp_maxpool" | head -5
SOL_STEM_POOL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stem_row_kernel -c 1 \
  -o gpurun_out/stem_pool_full -f python bench.py --steps 1 --warmup 1 --no-train --no-cpu-baseline --no-configs > gpurun_out/ncu_sp.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stem_row_kernel -c 1 \
  -o gpurun_out/stem_full -f python bench.py --steps 1 --warmup 1 --no-train --no-cpu-baseline --no-configs > gpurun_out/ncu_s.log 2>&1; echo "ncu rc=$?"
