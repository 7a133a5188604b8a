# gpurun recipe: cached bank searches -- parity + fusion tests, fused C1 passes, C1 bench per-op and fused
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fusion.py tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest_cache.log 2>&1
CFG=c1 timeout 300 python tools/fused_probe.py > gpurun_out/fused_c1.txt 2>&1
timeout 600 python bench.py --config c1 --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c1 --fuse --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c1_fuse.json 2> gpurun_out/bench_c1_fuse.err
