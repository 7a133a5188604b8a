# gpurun recipe: C3 per-regime times with parts of the gather_ws kernel disabled (HS_DEBUG_FLAGS:
# 1 no transform, 6 no loads/stores, 2 no loads, 4 no stores, 64 bulk rows off)
for f in 0 1 6 2 4 64 65 70; do
  echo "== flags $f" >> gpurun_out/phase_c3.txt
  HS_DEBUG_FLAGS=$f CFG=c3 LIMIT=40 timeout 300 python tools/ops_probe.py 2>&1 | tail -5 >> gpurun_out/phase_c3.txt
done
