# gpurun recipe: fusion equivalence tests, then fused C4 per-pass times: default vs dense tiles (bit 12) vs one-quad loop (bit 11)
timeout 600 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_graph.py -x -q > gpurun_out/pytest_fusion.log 2>&1; tail -3 gpurun_out/pytest_fusion.log
CFG=c4 N=15 timeout 600 python tools/fused_probe.py > gpurun_out/fused_c4_n15_new.txt 2>&1
HS_DEBUG_FLAGS=4096 CFG=c4 N=15 timeout 600 python tools/fused_probe.py > gpurun_out/fused_c4_n15_dense.txt 2>&1
sed -n 7,8p gpurun_out/fused_c4_n15_new.txt; sed -n 7,8p gpurun_out/fused_c4_n15_dense.txt
CFG=c4 N=17 timeout 900 python tools/fused_probe.py > gpurun_out/fused_c4_n17_new.txt 2>&1
sed -n 7,13p gpurun_out/fused_c4_n17_new.txt
CFG=c4 N=15 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 2 -c 1 \
  -f -o gpurun_out/c4_prog3 python tools/fused_probe.py > gpurun_out/ncu_prog.log 2>&1
