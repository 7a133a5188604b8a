# gpurun recipe: k=2 Kraus sums on the tensor-core gather -- parity, sharded, Kraus timings, C1 per-op
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py tests/test_gpu_graph.py tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_kraus.log 2>&1
timeout 600 python tools/kraus_probe.py > gpurun_out/kraus.txt 2>&1
CFG=c1 timeout 300 python tools/ops_probe.py 2>&1 | tail -7 > gpurun_out/ops_c1_tail.txt
