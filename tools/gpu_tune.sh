cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "overflow or redo" 2>&1 | tail -2
AB_CONFIGS="cfg3" bash tools/walk_ab.sh "" "-DBH_W9_FLUSH=16" "-DBH_W9_FLUSH=24" "-DBH_W9_PPFLUSH=48" "-DBH_W9_FULLMAX=32" "-DBH_BUCKET_UNROLL=4"
