# gpurun recipe: gather_ws bulk-row staging -- parity + sharded tests, per-op timings, C3/C1 bench
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_bulk.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1 or c3" >> gpurun_out/pytest_bulk.log 2>&1
CFG=c3 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c3.txt 2>&1
CFG=c1 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c1.txt 2>&1
for c in c3 c1; do timeout 400 python bench.py --config $c --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_${c}.json 2> gpurun_out/bench_${c}.err; done
