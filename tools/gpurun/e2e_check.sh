# gpurun recipe: C2 bench with the pipelined end-to-end measurement (plain and fused)
timeout 900 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c2e.json 2> gpurun_out/bench_c2e.err
timeout 900 python bench.py --no-cpu --steps 3 --warmup 3 --fuse > gpurun_out/bench_c2ef.json 2> gpurun_out/bench_c2ef.err
