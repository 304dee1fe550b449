cd $GRAFT_REPO_ROOT
python tools/repro_golden32.py 2>&1 | tail -2
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
