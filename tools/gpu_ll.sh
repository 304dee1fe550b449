cd $GRAFT_REPO_ROOT
for c in cfg3; do
python tools/step_cfg.py $c 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_$c.csv python tools/step_cfg.py $c 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/ll_$c.csv gpurun_out/ll_$c.json "$c one step" | head -40
done
