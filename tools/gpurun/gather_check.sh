# gpurun recipe: parity, fusion and sharded tests, then C3 and C1 benches (gather-kernel changes)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fusion.py tests/test_multigpu_gpu.py -x -q > gpurun_out/pytest_g.log 2>&1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1 or c3" >> gpurun_out/pytest_g.log 2>&1
for c in c3 c1; do timeout 400 python bench.py --config $c --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_${c}b.json 2> gpurun_out/bench_${c}b.err; done
