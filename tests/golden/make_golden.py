#!/usr/bin/env python3
"""Generate tests/golden/golden.npz by running the REFERENCE itself (arXiv 2604.15765, compiled from
/root/reference/proj/src by oracle/build_ref.sh, with the documented kernels.cpp:365/367/369 fix).

Each case: a seeded random hermitian operator (the reference's random_hermitian, storage.cpp:195-201),
one channel of the SPEC library (channel.cpp:82-154) plus Haar / random-Kraus generics, applied at a
target tuple chosen to exercise every tiled regime (intra, cross with subcases A/B/C, mixed, k = 3
dense fallback, n < m padding).  Stored: input payload, channel data, output payload, the
reference's ApplyPlan path and subcase counters.

    python tests/golden/make_golden.py      # needs /root/reference (this container only)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402


def haar(d, rng):
    z = (rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def kraus(k, r, rng):
    d = 1 << k
    z = (rng.normal(size=(r * d, d)) + 1j * rng.normal(size=(r * d, d))) / np.sqrt(2)
    q, _ = np.linalg.qr(z)
    return np.stack([q[a * d:(a + 1) * d] for a in range(r)])


def library(rng):
    ch = [O.native_gate(g) for g in "xyzsth"]
    ch.append(O.native_gate("rz", 0.7))
    ch.append(O.depolarising(0.1))
    ch.append(O.amplitude_damping(0.05))
    ch.append(O.generic(haar(2, rng), "haar1"))
    ch += [O.native_gate("cnot"), O.native_gate("swap")]
    ch.append(O.generic(haar(4, rng), "haar2"))
    ch.append(O.generic(kraus(2, 3, rng), "kraus2"))
    ch.append(O.native_gate("toffoli"))
    ch.append(O.generic(haar(8, rng), "haar3"))
    ch.append(O.generic(kraus(3, 2, rng), "kraus3"))
    return ch


TARGETS = {  # (n, m) -> k -> target tuples (constructor order)
    (5, 2): {1: [(0,), (1,), (2,), (4,)], 2: [(1, 0), (3, 2), (4, 2), (0, 3), (4, 1)], 3: [(0, 2, 4), (4, 3, 2), (1, 0, 3)]},
    (3, 5): {1: [(0,), (2,)], 2: [(2, 0)], 3: [(0, 1, 2)]},
    (6, 5): {1: [(5,)], 2: [(5, 0)], 3: [(5, 1, 3)]},
}


def main():
    ref = O.Reference()
    rng = np.random.default_rng(20260419)
    chans = library(rng)
    arrays, meta = {}, []
    for (n, m), tmap in TARGETS.items():
        h = ref.random_hermitian(n, 1000 + n, m)
        base = ref.view(h).copy()
        ref.free(h)
        arrays[f"in_{n}_{m}"] = base
        for ch in chans:
            if (n, m) == (6, 5) and ch.name not in ("h", "depolarising", "cnot", "haar2", "haar3", "kraus3"):
                continue  # keep the fixture small: the 48 KiB payload only for a few channels
            for tg in tmap.get(ch.k, []):
                h = ref.create(n, m, base)
                path, sub = ref.apply(h, ch, list(tg))
                out = ref.view(h).copy()
                ref.free(h)
                idx = len(meta)
                arrays[f"out_{idx}"] = out
                arrays[f"ops_{idx}"] = ch.ops
                meta.append({"n": n, "m": m, "name": ch.name, "kind": ch.kind, "targets": list(tg),
                             "phases": [[float(z.real), float(z.imag)] for z in ch.phases],
                             "perm": None if ch.perm is None else [int(v) for v in ch.perm],
                             "theta": ch.theta, "path": path, "subcases": list(sub)})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **arrays)
    print(f"wrote {out}: {len(meta)} cases, {os.path.getsize(out)} bytes")


if __name__ == "__main__":
    main()
