export KIFMM_PLAN_TIMING=1 KIFMM_TREE_TIMING=1
python tools/configs.py 2 2>&1 | grep -v "^{" | tail -40
python tools/configs.py 5 2>&1 | grep -v "^{" | tail -40
