# gpurun recipe: per-tile skew search -- parity (regimes, sharded), C3/C1 per-op timings
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest_skew.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1 or c3" >> gpurun_out/pytest_skew.log 2>&1
CFG=c3 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c3.txt 2>&1
CFG=c1 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c1.txt 2>&1
