# gpurun recipe: C2 headline -- launch list of bench.py --config c2 and ncu --set full of the pipe
# kernel applying depolarising(0.01) on qubit 10 (n = 16)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_c2_n16_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c2l.log 2>&1
CFG=c2 LIMIT=21 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 20 -c 1 \
  -o gpurun_out/r01_c2_n16_pipe_q10 python tools/ops_probe.py > gpurun_out/ncu_c2p.log 2>&1
