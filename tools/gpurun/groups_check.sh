# gpurun recipe: bulk mode with two copy groups -- parity (regimes, sharded), C3/C1 per-op timings
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest_grp.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1 or c3" >> gpurun_out/pytest_grp.log 2>&1
CFG=c3 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c3.txt 2>&1
HS_DEBUG_FLAGS=1 CFG=c3 LIMIT=40 timeout 300 python tools/ops_probe.py 2>&1 | tail -5 > gpurun_out/ops_c3_f1.txt
CFG=c1 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c1.txt 2>&1
