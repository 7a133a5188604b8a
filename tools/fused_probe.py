"""Diagnostics: per-pass launch times of one config's FUSED plan (CUDA events on the state's stream).
Run on a GPU box:  CFG=c1 python tools/fused_probe.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_15765_b200 import fusion  # noqa: E402
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

cfg = os.environ.get("CFG", "c1")
n = int(os.environ.get("N", {"c0": 12, "c1": 14, "c4": 17}.get(cfg, 16)))
m = 5
nat = H.nat
L = nat.engine()
st = H.TiledHermitian(n, m, device=0)
st.fill_mixture(HS.rank_psi(n, 3, 4))
ops = bench.build_ops(H, HS, cfg, n)
plan = fusion.plan_sequence([(spec, tg) for spec, tg, _ in ops], n, m)
opts = H.ApplyOptions(count_subcases=False)
ev = [ctypes.c_void_p() for _ in range(2 * len(plan.items))]
for e in ev:
    nat.check(L.hs_event_create(ctypes.byref(e)))
for _ in range(2):
    for i, item in enumerate(plan.items):
        L.hs_event_record(ev[2 * i], st.handle)
        fusion.execute(st, fusion.Plan([item]), opts)
        L.hs_event_record(ev[2 * i + 1], st.handle)
    st.synchronize()
for i, item in enumerate(plan.items):
    x = ctypes.c_float()
    nat.check(L.hs_event_elapsed_ms(ev[2 * i], ev[2 * i + 1], ctypes.byref(x)))
    if item[0] == "op":
        what = f"op {item[1].name} k={item[1].k} targets {item[2]} g={sum(1 for t in item[2] if t >= m)}"
    elif item[0] == "cxlayer":
        what = f"cxlayer pairs {item[1]}"
    else:
        what = f"{item[0]} qubits {[s.qubit for s in item[1]] if isinstance(item[1], list) else item[1].qubit}"
    print(f"{i:4d} {x.value:8.3f} ms  {what}")
