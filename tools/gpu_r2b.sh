cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "fp32_golden_tolerance" --tb=long 2>&1 | grep -v "^$" | tail -60
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15
