timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest15.log 2>&1
for c in c0 c1 c2; do timeout 400 python bench.py --config $c --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_${c}b.json 2> gpurun_out/bench_${c}b.err; done
