timeout 300 python scripts/profile_steps.py train 2>&1 | head -6
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('infer', d['value'], 'train', d['train']['value'], d['train']['ms_per_step'])"
timeout 900 python -m pytest tests/test_gpu_units.py tests/test_gpu_e2e.py tests/test_gpu_frontend.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x -k "train or composition or bench_train or transparent or context or bundle or running" 2>&1 | tail -2
