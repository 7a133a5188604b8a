# gpurun recipe: parity + fusion tests, C3 bench
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fusion.py -x -q > gpurun_out/pytest21.log 2>&1
timeout 400 python bench.py --config c3 --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.err
