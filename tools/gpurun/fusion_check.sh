# gpurun recipe: fusion equivalence tests and fused bench lines
timeout 300 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest19.log 2>&1
for c in c2 c0 c4; do timeout 600 python bench.py --config $c --fuse --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_${c}_fuse.json 2> gpurun_out/bench_${c}_fuse.err; done
