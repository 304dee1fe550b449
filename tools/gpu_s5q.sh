cd $GRAFT_REPO_ROOT
for f in "-DBH_W9_FCAP=96 -DBH_W9_CHECK=1" "-DBH_W9_PPSTAGE=1" "-DBH_W9_HALVES=1"; do
BH_NVCC_EXTRA="$f" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
echo "[$f]"; timeout 1200 python -m pytest tests/test_gpu_walk_schedules.py tests/test_gpu_walk_only.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x -k "walk or fp32 or scale or leaf or bucket or cfg" 2>&1 | tail -2
done
BH_NVCC_EXTRA="" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1
