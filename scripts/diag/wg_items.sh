for i in 1 2 3 4; do echo "items/SM=$i"; SOL_WG_ITEMS_PER_SM=$i python scripts/wgrad_micro.py; done
