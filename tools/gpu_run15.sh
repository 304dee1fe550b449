cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_decomposition.py -x -q 2>&1 | tail -3
AB_CONFIGS="cfg3 cfg2" bash tools/walk_ab.sh "" "-DBH_W9_PPFLUSH=40" "-DBH_W9_FLUSH=32" "-DBH_W9_FLUSH=32 -DBH_W9_PPFLUSH=48" "-DBH_BUCKET_UNROLL=2"
echo done
