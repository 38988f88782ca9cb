for v in 0 1; do
  if [ $v = 1 ]; then export SOL_DBG_SKIP_REPACK=1; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-configs --train-steps 20 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('skip_repack=$v train', d['train']['value'], d['train']['ms_per_step'])"
done
