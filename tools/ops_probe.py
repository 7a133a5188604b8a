"""Diagnostics: per-operation launch times of one config's op sequence (CUDA events on the state's
stream), grouped by grid-target count g.  Run on a GPU box:
    CFG=c3 [LIMIT=20] [HS_DEBUG_FLAGS=...] python tools/ops_probe.py [> gpurun_out/ops_c3.txt]"""
import ctypes
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

cfg = os.environ.get("CFG", "c3")
n = int(os.environ.get("N", {"c0": 12, "c1": 14, "c4": 17}.get(cfg, 16)))
m = 5
nat = H.nat
L = nat.engine()
st = H.TiledHermitian(n, m, device=0)
st.fill_mixture(HS.rank_psi(n, 3, 4))
ops = bench.build_ops(H, HS, cfg, n)[: int(os.environ.get("LIMIT", "100000"))]
opts = H.ApplyOptions(count_subcases=False)
ev = [ctypes.c_void_p() for _ in range(2 * len(ops))]
for e in ev:
    nat.check(L.hs_event_create(ctypes.byref(e)))
for _ in range(2):
    plans = []
    for i, (spec, tg, kind) in enumerate(ops):
        L.hs_event_record(ev[2 * i], st.handle)
        plans.append(H.apply(st, spec, tg, opts))
        L.hs_event_record(ev[2 * i + 1], st.handle)
    st.synchronize()
S = st.element_count() * 16
by = defaultdict(list)
for i, (spec, tg, kind) in enumerate(ops):
    x = ctypes.c_float()
    nat.check(L.hs_event_elapsed_ms(ev[2 * i], ev[2 * i + 1], ctypes.byref(x)))
    g = sum(1 for t in tg if t >= m)
    t = float(x.value)
    by[(kind, len(tg), g)].append(t)
    print(f"op {i:3d} {kind:8s} targets {str(tg):14s} g={g} path={plans[i].path:14s} {t:8.3f} ms "
          f"{plans[i].touched_bytes / t / 1e6:7.0f} GB/s")
print("summary (kind, k, g): count, mean ms, min, max, GB/s at 2S")
for key in sorted(by):
    v = by[key]
    mean = sum(v) / len(v)
    print(f"{key}: {len(v):3d}  {mean:8.3f}  {min(v):8.3f}  {max(v):8.3f}  {2 * S / mean / 1e6:7.0f}")
