cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x -k "fp32 or scale or leaf or bucket or cfg" 2>&1 | tail -2
AB_CONFIGS="cfg3 cfg4" bash tools/sort_ab.sh ""
