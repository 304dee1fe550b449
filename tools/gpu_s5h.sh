cd $GRAFT_REPO_ROOT
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_walk9" -s 1 -c 1 -o gpurun_out/walk_s5 python tools/step_cfg.py cfg3 1 > gpurun_out/walk_s5.log 2>&1
tail -2 gpurun_out/walk_s5.log
