# gpurun recipe: grid-program addressing -- fusion tests, fused C2 / C4 passes and bench lines
timeout 900 python -m pytest tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_prog2.log 2>&1
CFG=c4 timeout 600 python tools/fused_probe.py > gpurun_out/fused_c4.txt 2>&1
CFG=c2 timeout 600 python tools/fused_probe.py > gpurun_out/fused_c2.txt 2>&1
