for c in c3 c4; do timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --impl reference --config c3 --steps 1 --warmup 0 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err
