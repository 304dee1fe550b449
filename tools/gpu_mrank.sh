cd $GRAFT_REPO_ROOT
for d in distributed replicated; do
bash tools/mrank_smoke.sh 2 --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --decomp $d > gpurun_out/mr_$d.json 2> gpurun_out/mr_$d.err; echo "$d rc=$?"
tail -c 600 gpurun_out/mr_$d.json; tail -3 gpurun_out/mr_$d.err
done
BH_DIST_BACKEND=gloo BH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mr_spawn.json 2> gpurun_out/mr_spawn.err; echo "spawn rc=$?"; tail -c 300 gpurun_out/mr_spawn.json
timeout 600 python bench.py --gpus 2 --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mr_nogpu.json 2> gpurun_out/mr_nogpu.err; echo "2 gpus on 1: rc=$?"; tail -2 gpurun_out/mr_nogpu.err
