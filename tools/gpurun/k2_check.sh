# gpurun recipe: k=2 unitaries on one grid bit through the tensor-core gather -- parity, sharded, C1 bench
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_k2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1" >> gpurun_out/pytest_k2.log 2>&1
timeout 600 python bench.py --config c1 --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
