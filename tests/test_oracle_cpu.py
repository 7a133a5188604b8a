"""CPU tests of the oracle (test infrastructure) -- pinning it before it is trusted as the GPU checker.

1. against the golden vectors tests/golden/golden.npz, which the compiled REFERENCE produced
   (tests/golden/make_golden.py);
2. against the compiled reference itself (oracle/_ref/libhermsim_ref.so) on a sweep of sizes, tile
   exponents, channels and target tuples, including the kernel path and subcase counters;
3. against a naive dense Kraus oracle (SPEC.md reference_oracle: literal sum K H K^dagger);
4. the SPEC.md known-answer tests (insert_bits, tile_offset, footprints, depolarising, H, CNOT, <Z>, <X>);
5. the documented reference bug: the UNPATCHED tiled_two_mixed (kernels.cpp:365/367/369) is wrong on
   diagonal base pairs, the patched build is not.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


def _golden():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def _channel(O, rec, ops):
    ch = O.Channel(rec["name"], rec["kind"], np.ascontiguousarray(ops),
                   np.array([complex(a, b) for a, b in rec["phases"]]),
                   None if rec["perm"] is None else np.array(rec["perm"], np.uint32), rec["theta"])
    return ch


def test_golden_vectors_oracle(oracle, orc):
    z, meta = _golden()
    assert len(meta) >= 100
    for i, rec in enumerate(meta):
        n, m = rec["n"], rec["m"]
        base = z[f"in_{n}_{m}"]
        want = z[f"out_{i}"]
        got = base.copy()
        path, sub = orc.apply(got, n, m, _channel(oracle, rec, z[f"ops_{i}"]), rec["targets"])
        fro = orc.frobenius(want, n, m)
        assert oracle.rel_max_err(got, want, fro) <= 1e-14, (i, rec["name"], rec["targets"])
        assert path == rec["path"], (i, rec["name"], path, rec["path"])
        assert list(sub) == rec["subcases"], (i, rec["name"], sub, rec["subcases"])


def _haar(d, rng):
    z = (rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


@pytest.mark.parametrize("n,m", [(7, 2), (8, 5), (6, 0), (7, 3), (4, 5), (3, 5), (6, 1)])
def test_oracle_matches_reference(oracle, orc, ref, n, m):
    rng = np.random.default_rng(n * 31 + m)
    h = ref.random_hermitian(n, 77, m)
    base = ref.view(h).copy()
    ref.free(h)
    fro = orc.frobenius(base, n, m)
    chans = [oracle.native_gate(g) for g in "xyzsth"] + [
        oracle.native_gate("rz", 1.1), oracle.depolarising(0.2), oracle.amplitude_damping(0.3),
        oracle.generic(_haar(2, rng)), oracle.native_gate("cnot"), oracle.native_gate("swap"),
        oracle.generic(_haar(4, rng)), oracle.native_gate("toffoli"), oracle.generic(_haar(8, rng))]
    for ch in chans:
        k = ch.k
        if k > n:
            continue
        tlist = list(itertools.permutations(range(n), k))
        if len(tlist) > 40:
            tlist = [tlist[i] for i in rng.choice(len(tlist), 40, replace=False)]
        if k == 3 and n > 6:
            tlist = tlist[:4]
        for tg in tlist:
            a = base.copy()
            pa, sa = orc.apply(a, n, m, ch, list(tg))
            hh = ref.create(n, m, base)
            pb, sb = ref.apply(hh, ch, list(tg))
            b = ref.view(hh).copy()
            ref.free(hh)
            assert oracle.rel_max_err(a, b, fro) <= 1e-14, (ch.name, tg)
            assert pa == pb and sa == sb, (ch.name, tg, pa, pb, sa, sb)


def test_oracle_against_naive_dense_kraus(oracle, orc):
    """SPEC.md reference_oracle: out = sum K H K^dagger with dense triple loops (n <= 6)."""
    rng = np.random.default_rng(5)
    for n, m in ((5, 2), (6, 5), (4, 0)):
        d = (rng.normal(size=(1 << n, 1 << n)) + 1j * rng.normal(size=(1 << n, 1 << n)))
        dense = (d + d.conj().T) / 2
        base = orc.from_dense(dense, n, m)
        fro = orc.frobenius(base, n, m)
        for ch, tg in ((oracle.depolarising(0.1), (3,)), (oracle.native_gate("h"), (0,)),
                       (oracle.native_gate("cnot"), (3, 1)), (oracle.generic(_haar(4, rng)), (1, 3)),
                       (oracle.native_gate("toffoli"), (2, 0, 3)), (oracle.generic(_haar(8, rng)), (3, 0, 2)),
                       (oracle.amplitude_damping(0.2), (n - 1,)), (oracle.native_gate("y"), (2,))):
            got = base.copy()
            orc.apply(got, n, m, ch, list(tg))
            want = orc.from_dense(orc.dense_kraus_apply(dense, n, ch, list(tg)), n, m)
            assert oracle.rel_max_err(got, want, fro) <= 1e-13, (n, m, ch.name, tg)


def test_unpatched_reference_mixed_bug(oracle, orc, ref):
    """tiled_two_mixed writes wrong mirrors on diagonal base pairs; patched is correct."""
    try:
        bad = oracle.Reference(patched=False)
    except FileNotFoundError as e:
        pytest.skip(str(e))
    n, m = 7, 2
    rng = np.random.default_rng(9)
    h = ref.random_hermitian(n, 3, m)
    base = ref.view(h).copy()
    ref.free(h)
    fro = orc.frobenius(base, n, m)
    ch = oracle.generic(_haar(4, rng))
    tg = [5, 1]  # one target < m, one >= m: the mixed engine
    want = base.copy()
    path, _ = orc.apply(want, n, m, ch, tg)
    assert path == "tiled-mixed"
    outs = []
    for lib in (ref, bad):
        hh = lib.create(n, m, base)
        lib.apply(hh, ch, tg)
        outs.append(lib.view(hh).copy())
        lib.free(hh)
    assert oracle.rel_max_err(outs[0], want, fro) <= 1e-14
    assert oracle.rel_max_err(outs[1], want, fro) > 1e-6  # the published bug


# ------------------------------------------------------------------- SPEC known-answer tests
def test_spec_index_kats(orc, ref):
    for lib in (orc, ref):
        assert lib.insert_bits(0, 0, [0]) == 0
        assert lib.insert_bits(0, 1, [3]) == 8
        assert lib.insert_bits(5, 1, [1]) == 11
        assert lib.insert_bits(3, 3, [0, 2]) == 15
        assert lib.tile_offset(0, 0, 32) == 0
        assert lib.tile_offset(1, 0, 32) == 1024
        assert lib.tile_offset(2, 1, 32) == 4096
    # bijectivity of insert_bits over all (s, a) for A = {1, 4}, n = 6 (SPEC bit_index invariant)
    seen = {orc.insert_bits(s, a, [1, 4]) for s in range(16) for a in range(4)}
    assert seen == set(range(64))


def test_spec_footprint_kats(ref):
    from paper_2604_15765_b200.hermsim import footprint_bytes
    for n, want in ((3, 16384), (5, 16384), (10, 8650752)):
        assert ref.footprint_bytes(n, 5) == want
        assert footprint_bytes(n, 5) == want
    # SPEC.md Table I lists 16 KiB for n = 1, 2 at m = 5, but the reference's own validation
    # (storage.cpp:17-20, m <= n + 2) rejects those shapes; we follow the code, not the table.
    for n in (1, 2):
        assert ref.footprint_bytes(n, 5) == 0  # the reference threw std::invalid_argument
        with pytest.raises(ValueError):
            footprint_bytes(n, 5)
    assert abs(footprint_bytes(15, 5) / 2**30 - 8.0) < 0.01  # "8.0 GiB" (PAPER Table I)
    # tiled / dense = (N + M) / 2N exactly; the SPEC's "<= 0.502 for n >= 10" holds from n = 14
    # (n = 10 gives 0.5156), i.e. the "roughly halving" claim, not the printed bound
    for n in range(10, 26):
        assert footprint_bytes(n, 5) / (2 ** (2 * n) * 16) == 0.5 + 2.0 ** (5 - 1 - n)
        if n >= 14:
            assert footprint_bytes(n, 5) / (2 ** (2 * n) * 16) <= 0.502


def _projector(orc, n, m, b):
    d = np.zeros((1 << n, 1 << n), np.complex128)
    d[b, b] = 1.0
    return orc.from_dense(d, n, m)


def test_spec_channel_kats(oracle, orc):
    n, m = 1, 5
    p = _projector(orc, n, m, 0)
    orc.apply(p, n, m, oracle.depolarising(0.1), [0])
    dm = orc.to_dense(p, n, m)
    assert abs(dm[0, 0] - 14 / 15) < 1e-15 and abs(dm[1, 1] - 1 / 15) < 1e-15
    p = _projector(orc, n, m, 0)
    orc.apply(p, n, m, oracle.native_gate("h"), [0])
    assert np.allclose(orc.to_dense(p, n, m), 0.5, atol=1e-15)
    n = 2
    p = _projector(orc, n, m, 0b10)  # qubit 1 set
    orc.apply(p, n, m, oracle.native_gate("cnot"), [1, 0])  # control = first-listed target
    dm = orc.to_dense(p, n, m)
    assert dm[0b11, 0b11] == 1.0 and np.count_nonzero(dm) == 1


def test_spec_expectation_kats(oracle, orc):
    n, m = 1, 5
    rho = _projector(orc, n, m, 0)
    z = orc.from_dense(np.diag([1.0, -1.0]).astype(np.complex128), n, m)
    assert orc.expectation(rho, z, n, m) == 1.0  # <Z> on |0><0| = +1
    plus = orc.from_dense(np.full((2, 2), 0.5, np.complex128), n, m)
    x = orc.from_dense(np.array([[0, 1], [1, 0]], np.complex128), n, m)
    assert abs(orc.expectation(plus, x, n, m) - 1.0) < 1e-15  # <X> on |+><+| = +1


def test_expectation_strict_offdiagonal_bound(orc):
    """tr(rho O) with the strict ti > tj bound equals the dense trace."""
    rng = np.random.default_rng(2)
    for n, m in ((6, 2), (5, 5), (7, 3)):
        a = rng.normal(size=(1 << n, 1 << n)) + 1j * rng.normal(size=(1 << n, 1 << n))
        b = rng.normal(size=(1 << n, 1 << n)) + 1j * rng.normal(size=(1 << n, 1 << n))
        a, b = a + a.conj().T, b + b.conj().T
        got = orc.expectation(orc.from_dense(a, n, m), orc.from_dense(b, n, m), n, m)
        assert abs(got - np.trace(a @ b).real) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(b)


def test_subcase_closed_form(oracle, orc):
    """C = G/2, B = (G/2)(2^a' - 1)/2, A = P - B - C, P = (G/2)(G/2 + 1)/2."""
    n, m = 9, 3
    G = (1 << n) >> m
    base = np.zeros(oracle.payload_count(n, m), np.complex128)
    for a in range(m, n):
        ap = a - m
        _, (A, B, C) = orc.apply(base.copy(), n, m, oracle.depolarising(0.1), [a])
        P = (G // 2) * (G // 2 + 1) // 2
        assert C == G // 2 and B == (G // 2) * ((1 << ap) - 1) // 2 and A == P - B - C


def test_gaussian_entry_bit_exact(oracle, orc, ref):
    from paper_2604_15765_b200 import harness as HS
    for seed, c in ((0, 0), (7, 3), (2**63, 12345), (42, 2**40)):
        z = ref.gaussian_entry(seed, c)
        assert orc.gaussian_entry(seed, c) == z == HS.gaussian_entry(seed, c)
    assert math.isfinite(abs(z))
