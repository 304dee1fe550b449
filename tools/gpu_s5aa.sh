cd $GRAFT_REPO_ROOT
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_emit_mark|k_bucket_moments|k_emit_create|k_moments_coop|k_lcp_new|k_compact_parents|k_mom_lists" -s 7 -c 7 -o gpurun_out/build_s5 python tools/step_cfg.py cfg3 1 > gpurun_out/build_s5.log 2>&1
tail -2 gpurun_out/build_s5.log
