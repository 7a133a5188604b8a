set -x
timeout 600 python -m pytest tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest_mg.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 6 -c 2 -o gpurun_out/c3_gather python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c3l.log 2>&1
