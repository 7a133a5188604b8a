"""Diagnostics: permutation / Pauli ops (the pipe kernel's cycle walk) at n = 16, per regime."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

n = 16
st = H.TiledHermitian(n, 5)
st.fill_mixture(HS.rank_psi(n, 1, 4))
L = H.nat.engine()
ev = [ctypes.c_void_p() for _ in range(2)]
for e in ev:
    L.hs_event_create(ctypes.byref(e))
opts = H.ApplyOptions(count_subcases=False)
cx, x = H.native_gate("cnot"), H.native_gate("x")
for name, spec, tg in (("cx in,in", cx, [1, 3]), ("cx grid-ctl,in", cx, [9, 2]), ("cx in-ctl,grid", cx, [2, 9]),
                       ("cx grid,grid", cx, [12, 9]), ("x in", x, [3]), ("x grid", x, [11]),
                       ("swap in,grid", H.native_gate("swap"), [3, 11])):
    for rep in range(4):
        L.hs_event_record(ev[0], st.handle)
        plan = H.apply(st, spec, tg, opts)
        L.hs_event_record(ev[1], st.handle)
        st.synchronize()
        ms = ctypes.c_float()
        L.hs_event_elapsed_ms(ev[0], ev[1], ctypes.byref(ms))
    print(f"{name:16s} {tg}: {ms.value:.3f} ms, touched {plan.touched_bytes / 1e9:.2f} GB -> "
          f"{plan.touched_bytes / ms.value / 1e6:.0f} GB/s")
