# gpurun recipe: grid programs on TMA boxes -- fusion + parity tests, fused bench lines (C2, C4)
timeout 900 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_prog.log 2>&1
for c in c2 c4; do timeout 900 python bench.py --config $c --fuse --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_${c}_fuse.json 2> gpurun_out/bench_${c}_fuse.err; done
