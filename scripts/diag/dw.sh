timeout 600 python scripts/diag/mbv2_prof.py mobilenet_v2 2>&1 | grep -E "dwconv|total" | head -14
