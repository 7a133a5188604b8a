timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "parity or c3 or golden" > gpurun_out/pytest3.log 2>&1
timeout 600 python bench.py --config c3 --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.err
