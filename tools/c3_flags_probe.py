"""Diagnostics: C3-style k = 3 unitary launch times at n = 16 per grid-target regime with parts of the
warp-specialised gather switched off (HS_DEBUG_FLAGS: 1 = no transform, 2 = no loads, 4 = no
write-back), plus the SM clock sampled by nvidia-smi.  Run on a GPU box, one process per setting:
    for f in 0 1 6; do HS_DEBUG_FLAGS=$f python tools/c3_flags_probe.py; done"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

n = 16
nat = H.nat
L = nat.engine()
st = H.TiledHermitian(n, 5, device=0)
st.fill_mixture(HS.rank_psi(n, 3, 4))
spec = H.make_generic("u3", HS.haar(3, 7))
opts = H.ApplyOptions(count_subcases=False)
ev = [ctypes.c_void_p() for _ in range(2)]
for e in ev:
    nat.check(L.hs_event_create(ctypes.byref(e)))
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"],
                       stdout=subprocess.PIPE, text=True)
res = []
for tg in ([0, 2, 6], [1, 8, 12], [10, 15, 7]):
    for _ in range(3):
        H.apply(st, spec, tg, opts)
    st.synchronize()
    L.hs_event_record(ev[0], st.handle)
    reps = 20
    for _ in range(reps):
        H.apply(st, spec, tg, opts)
    L.hs_event_record(ev[1], st.handle)
    st.synchronize()
    x = ctypes.c_float()
    nat.check(L.hs_event_elapsed_ms(ev[0], ev[1], ctypes.byref(x)))
    res.append((tg, x.value / reps))
smi.terminate()
out = smi.communicate()[0].strip().splitlines()
clk = sorted(float(l.split(",")[0]) for l in out if l.strip())
pw = sorted(float(l.split(",")[1]) for l in out if l.strip())
flags = os.environ.get("HS_DEBUG_FLAGS", "0")
for tg, t in res:
    print(f"flags={flags} targets {str(tg):12s} {t:7.3f} ms  {68.753 / t:5.2f} TB/s")
print(f"flags={flags} sm clock median {clk[len(clk) // 2]:.0f} MHz  power median {pw[len(pw) // 2]:.0f} W")
