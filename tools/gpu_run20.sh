cd $GRAFT_REPO_ROOT
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_walk9" -s 1 -c 1 -o gpurun_out/walk3f python tools/step_cfg.py cfg3 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_sort_pass" -s 10 -c 1 -o gpurun_out/sort3f python tools/step_cfg.py cfg3 1 > /dev/null 2>&1
python tools/step_cfg.py cfg4 1 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_moments_coop|k_emit" -s 2 -c 2 -o gpurun_out/build4f python tools/step_cfg.py cfg4 1 > /dev/null 2>&1
echo done
