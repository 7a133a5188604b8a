# gpurun recipe: parity, C3 per-op timings and the C3 / C1 bench lines
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest_c3b.log 2>&1
CFG=c3 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c3.txt 2>&1
for c in c3 c1; do timeout 600 python bench.py --config $c --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_${c}.json 2> gpurun_out/bench_${c}.err; done
