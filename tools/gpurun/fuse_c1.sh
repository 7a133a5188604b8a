# gpurun recipe: composed same-target unitaries -- fusion tests, fused C1 bench line
timeout 900 python -m pytest tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_fc1.log 2>&1
timeout 600 python bench.py --config c1 --fuse --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c1_fuse.json 2> gpurun_out/bench_c1_fuse.err
