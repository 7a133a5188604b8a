# gpurun recipe: staging-mode parity tests, C3 per-op timings, DRAM bytes of the first three C3 gather launches
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "staging or library" > gpurun_out/pytest_promo.log 2>&1
CFG=c3 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c3.txt 2>&1
CFG=c3 LIMIT=3 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gather_ws -c 6 --csv --log-file gpurun_out/c3_dram.csv python tools/ops_probe.py > /dev/null 2>&1
