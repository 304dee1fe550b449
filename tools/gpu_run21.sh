cd $GRAFT_REPO_ROOT
AB_CONFIGS="cfg3 cfg4" bash tools/sort_ab.sh "" "-DBH_SORT_VIDX=1 -DBH_SORT_BLOCKS=4" "-DBH_SORT_VIDX=1"
BH_DIST_BACKEND=gloo BH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gpus2.json 2> gpurun_out/gpus2.err; echo gpus2 rc=$?
tail -c 600 gpurun_out/gpus2.json; tail -3 gpurun_out/gpus2.err
echo done
