cd $GRAFT_REPO_ROOT
timeout 300 python tools/c3_probe.py 100 > gpurun_out/c3_live.log 2>&1 || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,smsp__inst_executed.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/c3_probe.py 2 > gpurun_out/c3_ncu.log 2>&1
cat gpurun_out/c3_live.log
