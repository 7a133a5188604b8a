# gpurun recipe: k=2 unitaries through the tensor-core gather -- parity, sharded, fusion, C1 per-op + bench
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py tests/test_gpu_fusion.py tests/test_gpu_graph.py -x -q > gpurun_out/pytest_k2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1" >> gpurun_out/pytest_k2.log 2>&1
CFG=c1 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c1.txt 2>&1
timeout 600 python bench.py --config c1 --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
