# gpurun recipe: parity (incl. staging modes), C3 bench, C4 / C2 per-op timings
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "not c4" > gpurun_out/pytest_nli.log 2>&1
timeout 600 python bench.py --config c3 --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
CFG=c4 timeout 600 python tools/ops_probe.py > gpurun_out/ops_c4.txt 2>&1
CFG=c2 timeout 300 python tools/ops_probe.py > gpurun_out/ops_c2.txt 2>&1
