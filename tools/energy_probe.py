"""Diagnostics: energy per operation (NVML total-energy counter) and SM clock for representative
n = 16 operations: is a config power-capped?  Run on a GPU box: python tools/energy_probe.py"""
import os
import sys
import time

import pynvml

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402

n = int(os.environ.get("N", "16"))
reps = int(os.environ.get("REPS", "20"))
pynvml.nvmlInit()
dev = pynvml.nvmlDeviceGetHandleByIndex(0)
st = H.TiledHermitian(n, 5, device=0)
st.fill_mixture(HS.rank_psi(n, 3, 4))
opts = H.ApplyOptions(count_subcases=False)
S = st.element_count() * 16
cases = [
    ("depolarising q10 (pipe)", H.depolarising(0.01), [10]),
    ("hadamard q2 (pipe)", H.native_gate("h"), [2]),
    ("haar3 [0,2,6] g=1", H.make_generic("u3", HS.haar(3, 7)), [0, 2, 6]),
    ("haar3 [2,9,13] g=2", H.make_generic("u3", HS.haar(3, 7)), [2, 9, 13]),
    ("haar3 [5,11,13] g=3", H.make_generic("u3", HS.haar(3, 7)), [5, 11, 13]),
]
for name, spec, tg in cases:
    H.apply(st, spec, tg, opts)
    st.synchronize()
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(dev)
    t0 = time.perf_counter()
    clk = []
    for r in range(reps):
        H.apply(st, spec, tg, opts)
        if r % 4 == 3:
            clk.append(pynvml.nvmlDeviceGetClockInfo(dev, pynvml.NVML_CLOCK_SM))
    st.synchronize()
    dt = time.perf_counter() - t0
    e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(dev)
    joule = (e1 - e0) * 1e-3 / reps
    print(f"{name:26s} {dt / reps * 1e3:7.2f} ms/op  {joule:6.2f} J/op  {joule / (dt / reps):6.0f} W  "
          f"{2 * S / (dt / reps) / 1e9:6.0f} GB/s  sm {sorted(clk)[len(clk) // 2]} MHz")
