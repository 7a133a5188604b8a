# gpurun recipe: DRAM bytes per launch (ncu, one metric pass) of the first C1 and C4 operations
CFG=c1 LIMIT=4 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/c1_dram.csv python tools/ops_probe.py > gpurun_out/c1_dram.log 2>&1
CFG=c4 LIMIT=3 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/c4_dram.csv python tools/ops_probe.py > gpurun_out/c4_dram.log 2>&1
