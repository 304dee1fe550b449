cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2
AB_CONFIGS="cfg3" bash tools/walk_ab.sh ""
bash tools/mrank_smoke.sh 2 --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --decomp replicated > gpurun_out/mr_r.json 2> gpurun_out/mr_r.err; echo "mrank rc=$?"
