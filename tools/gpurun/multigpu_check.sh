# gpurun recipe: sharded engine (P shards on one GPU) against the single-GPU engine, parity suite
timeout 600 python -m pytest tests/test_multigpu_gpu.py tests/test_gpu_parity.py tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_mg.log 2>&1
timeout 400 python bench.py --config c2 --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c2x.json 2> gpurun_out/bench_c2x.err
