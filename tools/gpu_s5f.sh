cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for e in "BH_ORDER_OVERLAP=1" "BH_ORDER_OVERLAP=0"; do AB_CONFIGS="cfg3 cfg2" bash tools/env_ab.sh "$e"; done
