# maxpool band-kernel sweep: per-step times of the inference plan for band height R / blocks per SM
for cfg in "0 2" "1 1" "1 2" "1 3" "2 1" "2 2"; do
  set -- $cfg
  echo "R=$1 BPS=$2"; SOL_POOL_BAND=$1 SOL_POOL_BPS=$2 timeout 300 python scripts/profile_steps.py infer fuse 2>&1 | grep -E "^total|^dfp_maxpool"
done
timeout 600 python -m pytest tests/test_gpu_units.py tests/test_gpu_e2e.py -q -m gpu -p no:cacheprovider -k "small_cnn or resnet or stem" 2>&1 | tail -2
