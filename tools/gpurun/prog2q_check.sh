# gpurun recipe: fusion equivalence tests (short timeouts: barrier protocols), then fused C4 per-pass times: default vs lockstep loop (bit 11)
timeout 300 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_graph.py tests/test_gpu_races.py -x -q > gpurun_out/pytest_fusion.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fusion.log
CFG=c4 N=15 timeout 120 python tools/fused_probe.py > gpurun_out/fused_c4_n15_new.txt 2>&1; echo "probe rc=$?"
HS_DEBUG_FLAGS=2048 CFG=c4 N=15 timeout 120 python tools/fused_probe.py > gpurun_out/fused_c4_n15_lock.txt 2>&1
sed -n 7,8p gpurun_out/fused_c4_n15_new.txt; sed -n 7,8p gpurun_out/fused_c4_n15_lock.txt
CFG=c4 N=17 timeout 300 python tools/fused_probe.py > gpurun_out/fused_c4_n17_new.txt 2>&1
sed -n 1,13p gpurun_out/fused_c4_n17_new.txt
