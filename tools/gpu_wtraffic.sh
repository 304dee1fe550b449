cd $GRAFT_REPO_ROOT
for c in cfg2 cfg3 cfg4; do
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_walk9 -c 1 --csv --log-file gpurun_out/wt_$c.csv python tools/step_cfg.py $c 0 > /dev/null 2>&1
echo $c; grep -E "dram__bytes|pipe_fma" gpurun_out/wt_$c.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
