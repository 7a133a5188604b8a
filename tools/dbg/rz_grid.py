"""Diagnostics: Rz on a grid qubit (C4's slowest per-op kind) at n = 16, timed per launch."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

n = int(os.environ.get("N", "16"))
q = int(os.environ.get("Q", "10"))
st = H.TiledHermitian(n, 5)
st.fill_mixture(HS.rank_psi(n, 1, 4))
L = H.nat.engine()
ev = [ctypes.c_void_p() for _ in range(2)]
for e in ev:
    L.hs_event_create(ctypes.byref(e))
opts = H.ApplyOptions(count_subcases=False)
for name, spec in (("rz", H.native_gate("rz", 0.7)), ("depol", H.depolarising(0.01)), ("h", H.native_gate("h"))):
    for rep in range(4):
        L.hs_event_record(ev[0], st.handle)
        plan = H.apply(st, spec, [q], opts)
        L.hs_event_record(ev[1], st.handle)
        st.synchronize()
        ms = ctypes.c_float()
        L.hs_event_elapsed_ms(ev[0], ev[1], ctypes.byref(ms))
    print(f"{name} q={q} n={n}: {ms.value:.3f} ms, touched {plan.touched_bytes / 1e9:.2f} GB -> "
          f"{plan.touched_bytes / ms.value / 1e6:.0f} GB/s")
