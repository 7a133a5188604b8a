"""Diagnostics: one C4 CX layer (n from N, default 15) for ncu:
    ncu --set full -k regex:cx_layer python tools/cx_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

n = int(os.environ.get("N", "15"))
st = H.TiledHermitian(n, 5)
st.fill_mixture(HS.rank_psi(n, 3, 4))
pairs, _ = HS.matching_c4(n, HS.SEEDS["c4"] + 31)
for _ in range(3):
    H.apply_cx_layer(st, pairs)
st.synchronize()
print("pairs", pairs)
