timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest4.log 2>&1
for c in c3 c1; do timeout 600 python bench.py --config $c --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_${c}b.json 2> gpurun_out/bench_${c}b.err; done
