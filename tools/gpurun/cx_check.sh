# gpurun recipe: CX layers -- bit-identity and fusion tests, fused C4 passes and bench line
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_cx.log 2>&1
CFG=c4 timeout 600 python tools/fused_probe.py > gpurun_out/fused_c4.txt 2>&1
timeout 900 python bench.py --config c4 --fuse --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c4_fuse.json 2> gpurun_out/bench_c4_fuse.err
