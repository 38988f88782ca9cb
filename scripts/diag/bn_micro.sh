echo default; python scripts/diag/bn_micro.py
echo no_coop; SOL_NO_COOP_FINALIZE=1 python scripts/diag/bn_micro.py
echo no_bulk; SOL_NO_BULK_REDUCE=1 python scripts/diag/bn_micro.py
