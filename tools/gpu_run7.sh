cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -rs 2>&1 | tail -5
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_sort_hist" -s 1 -c 1 -o gpurun_out/hist python tools/step_cfg.py cfg3 1 > /dev/null 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2203_08966_b200.engine import Engine
e=Engine('fp64',0); print('dfma', e.ffma_peak_tflops(True), 'ffma', e.ffma_peak_tflops(False))"
echo done
