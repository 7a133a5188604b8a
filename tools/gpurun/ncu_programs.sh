# gpurun recipe: ncu captures of one fused C4 grid program (9 chained steps) and one in-tile program (15 steps) at n=15
CFG=c4 N=15 timeout 600 python tools/fused_probe.py > gpurun_out/fused_c4_n15.txt 2>&1
CFG=c4 N=15 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_ws -s 4 -c 1 \
  -f -o gpurun_out/c4_gprog python tools/fused_probe.py > gpurun_out/ncu_gprog.log 2>&1
CFG=c4 N=15 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 1 -c 1 \
  -f -o gpurun_out/c4_prog python tools/fused_probe.py > gpurun_out/ncu_prog.log 2>&1
tail -3 gpurun_out/ncu_gprog.log gpurun_out/ncu_prog.log; head -14 gpurun_out/fused_c4_n15.txt
