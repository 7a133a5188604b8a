# gpurun recipe: smoke, GPU tests, all bench configs (per-op with e2e + CPU reference; fused), C3 launch
# list and ncu captures of the gather_ws variants (g=1 bulk rows, g=2 TMA boxes by quadrant, g=3 TMA boxes)
set -x
mkdir -p gpurun_out/r01_bench
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01_bench/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01_bench/pytest_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/r01_bench/bench_c2.json 2> gpurun_out/r01_bench/bench_c2.err
for c in c0 c1 c3 c4; do timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/r01_bench/bench_$c.json 2> gpurun_out/r01_bench/bench_$c.err; done
for c in c2 c0 c1 c4; do timeout 900 python bench.py --config $c --fuse --no-e2e --no-cpu --steps 3 --warmup 3 > gpurun_out/r01_bench/bench_${c}_fused.json 2> gpurun_out/r01_bench/bench_${c}_fused.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_c3_n16_launches.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c3l.log 2>&1
CFG=c3 LIMIT=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_ws -s 0 -c 3 \
  -o gpurun_out/r01_c3_gather_ws_variants python tools/ops_probe.py > gpurun_out/ncu_c3v.log 2>&1
