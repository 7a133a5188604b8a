"""Diagnostics: launch times of generic Kraus channels (rank > 1) at n = 16, k = 1, 2, 3, per grid-target
count.  Run on a GPU box: python tools/kraus_probe.py"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

n = int(os.environ.get("N", "16"))
nat = H.nat
L = nat.engine()
st = H.TiledHermitian(n, 5, device=0)
st.fill_mixture(HS.rank_psi(n, 3, 4))
opts = H.ApplyOptions(count_subcases=False)
S = st.element_count() * 16


def kraus(k, r, seed):
    rng = np.random.default_rng(seed)
    d = 1 << k
    a = rng.normal(size=(r * d, d)) + 1j * rng.normal(size=(r * d, d))
    q, _ = np.linalg.qr(a)
    return q.reshape(r, d, d)


cases = [(1, [3]), (1, [9]), (2, [1, 3]), (2, [3, 4]), (2, [2, 9]), (2, [9, 2]), (2, [8, 12]), (2, [14, 15]),
         (3, [0, 2, 4]), (3, [1, 3, 9]), (3, [2, 8, 12]), (3, [6, 9, 13])]
ranks = {1: (2, 4), 2: tuple(int(x) for x in os.environ.get("RANKS2", "2,4,16").split(",")),
         3: tuple(int(x) for x in os.environ.get("RANKS3", "2,4").split(","))}
reps = int(os.environ.get("REPS", "3"))
ev = [ctypes.c_void_p() for _ in range(2)]
for e in ev:
    nat.check(L.hs_event_create(ctypes.byref(e)))
for k, tg in cases:
    for r in ranks[k]:
        spec = H.make_generic(f"kraus{k}_{r}", kraus(k, r, 10 * k + r))
        H.apply(st, spec, tg, opts)
        st.synchronize()
        L.hs_event_record(ev[0], st.handle)
        for _ in range(reps):
            plan = H.apply(st, spec, tg, opts)
        L.hs_event_record(ev[1], st.handle)
        st.synchronize()
        x = ctypes.c_float()
        nat.check(L.hs_event_elapsed_ms(ev[0], ev[1], ctypes.byref(x)))
        t = x.value / reps
        print(f"k={k} rank={r:2d} targets {str(tg):12s} path={plan.path:14s} {t:8.3f} ms  "
              f"{2 * S / t / 1e6:7.0f} GB/s at 2S", flush=True)
