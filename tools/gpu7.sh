for f in 2 4 6 1; do HS_DEBUG_FLAGS=$f timeout 600 python bench.py --config c3 --no-e2e --no-cpu --steps 1 --warmup 1 > gpurun_out/bench_c3f$f.json 2>&1; done
