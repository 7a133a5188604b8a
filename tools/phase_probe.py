"""Diagnostics: per-phase cycles of the gather kernel (HS_DEBUG_FLAGS bit 4) for k = 3 unitaries at
n = 16, one op per grid-bit regime.  Run on a GPU box: HS_DEBUG_FLAGS=16 python tools/phase_probe.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

n = int(os.environ.get("N", "16"))
L = H.nat.engine()
L.hs_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
st = H.TiledHermitian(n, 5, device=0)
st.fill_mixture(HS.rank_psi(n, 3, 4))
spec = H.make_generic("u3", HS.haar(3, 7))
opts = H.ApplyOptions(count_subcases=False)
out = (ctypes.c_ulonglong * 8)()
for tg in ([10, 12, 14], [2, 9, 13], [0, 1, 9], [3, 6, 11]):
    for rep in range(3):
        L.hs_debug_phase_cycles(out)
        st.synchronize()
        t0 = time.perf_counter()
        H.apply(st, spec, tg, opts)
        st.synchronize()
        dt = time.perf_counter() - t0
        L.hs_debug_phase_cycles(out)
    v = list(out)
    tot = [v[q] + v[4 + q] for q in range(4)]
    s = sum(tot) or 1
    print(f"targets {tg}: {dt * 1e3:.2f} ms  wait {tot[0] / s:.1%}  transform {tot[1] / s:.1%}  "
          f"writeback {tot[2] / s:.1%}  load {tot[3] / s:.1%}  (cycles per CTA-group {s / 296:.3e})")
