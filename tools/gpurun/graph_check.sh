# gpurun recipe: CUDA-graph replay in bench (C0 n=12; C2 at n=10 where launches are short)
for a in "" "--graph"; do
  timeout 300 python bench.py --config c0 --no-e2e --no-cpu --steps 20 --warmup 3 $a > gpurun_out/graph_c0$a.json 2>&1
  timeout 300 python bench.py --config c2 --qubits 10 --no-e2e --no-cpu --steps 20 --warmup 3 $a > gpurun_out/graph_c2n10$a.json 2>&1
done
