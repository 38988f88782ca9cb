timeout 300 python scripts/profile_steps.py train family=dfp_pointwise 2>&1 | tail -102 | head -45
timeout 300 python scripts/profile_steps.py train family=bn_back_x 2>&1 | tail -54 | head -20
