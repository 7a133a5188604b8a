# gpurun recipe: ncu --set full of the first three C3 gather_ws launches (g=1 bulk, g=2 bulk, g=3 cp.async)
CFG=c3 LIMIT=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_ws -s 0 -c 3 \
  -o gpurun_out/r01_c3_gather_ws_regimes python tools/ops_probe.py > gpurun_out/ncu_c3_regimes.log 2>&1
