timeout 300 python scripts/profile_steps.py train 2>&1 | head -30
timeout 300 python scripts/profile_steps.py train family=conv_wgrad_tcgen05 2>&1 | tail -55
