HS_DEBUG_FLAGS=1 timeout 600 python bench.py --config c3 --no-e2e --no-cpu --steps 1 --warmup 1 > gpurun_out/bench_c3nc.json 2>&1
timeout 1100 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 6 -c 1 -o gpurun_out/c3_gather4 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c3d.log 2>&1
