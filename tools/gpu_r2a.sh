cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b3.json 2>gpurun_out/b3.err; tail -c 3000 gpurun_out/b3.json
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2.json 2>gpurun_out/b2.err; tail -c 3000 gpurun_out/b2.json
python -c "import __graft_entry__ as g; g.smoke()"
echo done
