for v in 1 0 1 0; do
SOL_PDL=$v timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-configs --no-train > gpurun_out/pdl_$v.log 2>&1; echo "pdl=$v rc=$?"
tail -1 gpurun_out/pdl_$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pdl=$v infer', round(d['value']), d['ms_per_step'])" 2>&1 | tail -1
done
