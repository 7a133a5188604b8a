"""Every kernel instantiation of the engine at small n: the race / synchronisation stress driver.

compute-sanitizer is closed on this GPU pool ("runs under it have left GPUs needing a reset"), so
races and barrier bugs are hunted by perturbation instead (tests/test_gpu_races.py runs this script
under each setting and requires the same SHA-256 digest of every result, plus oracle parity):
  HS_DEBUG_FLAGS=1024   every ring stage is NaN-filled between its write-back and its next load, so
                        a transform that reads before the copies landed, or a write-back that reads
                        after the refill started, leaves NaN in the result;
  HS_DEBUG_GRID=g       g persistent CTAs instead of one per SM: items move between CTAs and the
                        per-CTA item order changes.
Where compute-sanitizer is available the same script is its workload:

  compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_cases.py

Covers: pipe_kernel (k = 1 transfer / Hadamard / monomials incl. the compacted and grouped tile
permutations, k = 2 transfer on the pipe when m < 5, programs), gather_ws_kernel (k = 3 unitaries in
every staging mode: bulk rows, TMA boxes with and without quadrants, 4-tile items, cp.async for m < 5;
k = 2 unitaries through the pairing and the promotions; k = 2 Kraus sums in S form on whole tiles,
mixed and cross units; k = 3 Kraus sums of rank 2..4; grid programs), gather_kernel and conj_kernel
(k = 3 Kraus sums of rank > 4, k = 2 transfer matrices for m < 5, diagonal units), cx_layer_kernel,
reductions, device generators, format conversions, and peer-mode sharded ops (ShardGroup, one process).
Each case also checks its result against the CPU oracle, so a sanitizer run doubles as a parity run.
"""
import hashlib
import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402  (test infrastructure: the checker)
from paper_2604_15765_b200 import fusion  # noqa: E402
from paper_2604_15765_b200 import harness as HS  # noqa: E402
from paper_2604_15765_b200 import hermsim as H  # noqa: E402
from paper_2604_15765_b200.multigpu import ShardGroup  # noqa: E402

orc = O.Oracle()
worst = 0.0
count = 0
DIGEST = hashlib.sha256()


def digest(arr):
    DIGEST.update(np.ascontiguousarray(arr).view(np.uint8).tobytes())


def kraus(k, r, seed):
    rng = np.random.default_rng(seed)
    d = 1 << k
    z = (rng.normal(size=(r * d, d)) + 1j * rng.normal(size=(r * d, d))) / np.sqrt(2)
    q, _ = np.linalg.qr(z)
    return np.stack([q[a * d:(a + 1) * d, :] for a in range(r)])


def check(st, spec, och, n, m, tg, base):
    global worst, count
    want = base.copy()
    orc.apply(want, n, m, och, list(tg))
    st.upload(base)
    H.apply(st, spec, list(tg))
    got = st.download()
    digest(got)
    err = O.rel_max_err(got, want, orc.frobenius(base, n, m))
    worst = max(worst, err)
    count += 1
    if err > 1e-12:
        raise SystemExit(f"parity failure {spec.name} {tg} n={n} m={m}: {err}")


def channels():
    u1, u2, u3 = HS.haar(1, 1), HS.haar(2, 2), HS.haar(3, 3)
    out = [(H.native_gate(g), O.native_gate(g)) for g in ("h", "x", "y", "z", "t", "cnot", "swap", "toffoli")]
    out += [(H.native_gate("rz", 0.4), O.native_gate("rz", 0.4)), (H.depolarising(0.1), O.depolarising(0.1)),
            (H.amplitude_damping(0.2), O.amplitude_damping(0.2)), (H.make_generic("u1", u1), O.generic(u1)),
            (H.make_generic("u2", u2), O.generic(u2)), (H.make_generic("u3", u3), O.generic(u3)),
            (H.dual_channel(H.make_generic("u3", u3)), O.dual(O.generic(u3)))]
    for k, r in ((1, 3), (2, 2), (2, 16), (3, 2), (3, 4), (3, 6)):
        ks = kraus(k, r, 10 * k + r)
        out.append((H.make_generic(f"k{k}r{r}", ks), O.generic(ks)))
    return out


def main():
    for n, m in ((10, 5), (9, 5), (8, 3), (7, 2)):
        psi = HS.rank_psi(n, 5 + n, 4)
        base = HS.rho_payload(n, psi, m)
        st = H.TiledHermitian(n, m)
        for spec, och in channels():
            k = spec.k
            pool = list(itertools.permutations(range(n), k))
            rng = np.random.default_rng(n * 100 + m + k)
            picks = [pool[i] for i in rng.choice(len(pool), size=min(len(pool), {1: 6, 2: 8, 3: 8}[k]), replace=False)]
            if k == 3 and n == 10 and m == 5:  # every staging mode (tests/test_gpu_parity.py STAGING_CASES)
                picks += [(0, 2, 4), (4, 1, 3), (0, 2, 6), (6, 4, 1), (1, 6, 8), (9, 2, 5), (3, 6, 8), (9, 7, 5)]
            if k == 2 and n == 10 and m == 5:
                picks += [(1, 3), (3, 4), (2, 9), (9, 2), (6, 8), (9, 5)]
            for tg in picks:
                check(st, spec, och, n, m, tg, base)
        # fused programs (in-tile program, grid programs) and the CX layer
        seq = [(H.depolarising(0.01) if op.kind == "depol" else H.amplitude_damping(0.05), list(op.targets))
               for op in HS.config_ops("c2", n)]
        plan = fusion.plan_sequence(seq, n, m)
        st.upload(base)
        fusion.execute(st, plan)
        H.apply_cx_layer(st, [(0, n - 1), (2, 3), (n - 2, 1)])
        digest(st.download())
        # reductions and generators
        st.fill_mixture(psi)
        obs = H.TiledHermitian(n, m)
        obs.fill_pauli_sum(*HS.pauli_strings(n, 16, 3))
        digest(np.array([H.expectation(st, obs), H.trace(st), H.frobenius(st)]))
        obs.fill_random_hermitian(7)
        obs.fill_basis_projector(3)
        # format conversions (to_dense / convert, storage.cpp:241-292)
        dense = obs.to_dense()
        obs.from_dense(dense)
        obs.from_packed(obs.to_packed())
        rt = H.convert(obs, "tiled", max(0, m - 2))
        digest(dense)
        digest(rt.download())
        rt.free()
        obs.free()
        st.free()
    # sharded, peer mode and exchange mode (one process, one GPU)
    for peer in (False, True):
        n = 10
        grp = ShardGroup(n, 5, 4, peer=peer)
        grp.fill_mixture(HS.rank_psi(n, 42, 4))
        for spec, tg in ((H.native_gate("h"), [9]), (H.make_generic("u3", HS.haar(3, 4)), [9, 8, 1]),
                         (H.native_gate("cnot"), [9, 8]), (H.make_generic("k2", kraus(2, 2, 5)), [9, 2]),
                         (H.depolarising(0.1), [8])):
            grp.apply(spec, tg)
        grp.synchronize()
        for sh in grp.shards:
            digest(sh.download())
        grp.free()
    print(f"sanitize_cases: {count} checked cases, worst rel err {worst:.3e}")
    print(f"DIGEST {DIGEST.hexdigest()}")


if __name__ == "__main__":
    main()
