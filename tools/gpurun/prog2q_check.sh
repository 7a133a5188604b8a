# gpurun recipe: fusion equivalence tests, fused C4 per-pass times, fused bench lines
timeout 600 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_graph.py tests/test_gpu_races.py -x -q > gpurun_out/pytest_fusion.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fusion.log
CFG=c4 N=17 timeout 300 python tools/fused_probe.py > gpurun_out/fused_c4_n17_new.txt 2>&1
sed -n 1,13p gpurun_out/fused_c4_n17_new.txt
CFG=c2 N=16 timeout 300 python tools/fused_probe.py > gpurun_out/fused_c2_n16_new.txt 2>&1
cat gpurun_out/fused_c2_n16_new.txt
for c in c4 c2; do timeout 900 python bench.py --config $c --fuse --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_${c}_fuse.json 2> gpurun_out/bench_${c}_fuse.err; cat gpurun_out/bench_${c}_fuse.json; done
