"""Diagnostics: three k = 3 unitaries (one per grid-target regime) at n = 10 -- a seconds-long
check that a new gather-kernel build runs to completion before longer GPU jobs (run it under
`timeout`; e.g. after register-allocation changes such as setmaxnreg, where an unbalanced split
hangs the kernel)."""
import sys; sys.path.insert(0,'.')
from paper_2604_15765_b200 import harness as HS, hermsim as H
n=10
st=H.TiledHermitian(n,5); st.fill_mixture(HS.rank_psi(n,3,4))
for tg in ([0,2,6],[1,8,7],[9,5,7]):
    H.apply(st, H.make_generic("u3", HS.haar(3,7)), tg); st.synchronize(); print("ok", tg, flush=True)
