cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:"k_emit_mark" -c 1 -o gpurun_out/emitmark python tools/step_cfg.py cfg3 0 > /dev/null 2>&1; echo done
