# gpurun recipe: sharded engine (P shards on one GPU) against the single-GPU engine
timeout 600 python -m pytest tests/test_multigpu_gpu.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_mg.log 2>&1
