cd $GRAFT_REPO_ROOT
BH_DIST_BACKEND=gloo BH_SHARE_GPU=1 BH_DIST_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29533 tools/dist_profile.py cfg3 > gpurun_out/dist8_cfg3.txt 2>&1; echo rc=$?
head -60 gpurun_out/dist8_cfg3.txt
python tools/step_cfg.py cfg4 1 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_moments_coop" -s 1 -c 1 -o gpurun_out/mom4 python tools/step_cfg.py cfg4 1 > /dev/null 2>&1
echo done
