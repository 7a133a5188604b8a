# gpurun recipe: in-tile k=3 on the 12-stage gather -- parity (staging modes, library), C3 per-op timings
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest_g0.log 2>&1
CFG=c3 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c3.txt 2>&1
