# gpurun recipe: ncu capture of one fused C4 grid program (kind-0 steps) at n=15
CFG=c4 N=15 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_ws -s 0 -c 1 \
  -o gpurun_out/c4_gprog python tools/fused_probe.py > gpurun_out/ncu_gprog.log 2>&1
