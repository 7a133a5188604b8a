"""Size-independent properties of the hot path on the GPU (SPEC.md's intended strategy, SURVEY 4:
duality `SPEC.md:473,586`, hermiticity / trace drift `:346-347,585`, run-to-run determinism
`:358,590`), at small sizes for every channel kind and at config sizes (n = 14, n = 16) where no CPU
result is needed:

* duality: tr(E(rho) O) = tr(rho E^dagger(O)) with E^dagger = dual_channel(E)
  (/root/reference/proj/src/channel.cpp:188-194);
* a trace-preserving sequence keeps tr(rho) = 1 and the stored diagonal tiles hermitian
  (the mirror halves the reference keeps in sync, native.cpp:442-446, kernels.cpp:285-297);
* linearity: E(a X + b Y) = a E(X) + b E(Y) to rounding;
* the same sequence applied twice from the same input gives bit-identical payloads.
"""
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def H():
    from paper_2604_15765_b200 import hermsim
    if hermsim.device_count() < 1:
        pytest.fail("no CUDA device visible")
    return hermsim


@pytest.fixture(scope="module")
def HS():
    from paper_2604_15765_b200 import harness
    return harness


def _kraus(k, r, seed):
    """Random CPTP Kraus set: blocks of a Haar isometry."""
    rng = np.random.default_rng(seed)
    d = 1 << k
    z = (rng.normal(size=(r * d, d)) + 1j * rng.normal(size=(r * d, d))) / np.sqrt(2)
    q, _ = np.linalg.qr(z)
    return np.stack([q[a * d:(a + 1) * d, :] for a in range(r)])


def _channels(H, HS):
    out = [(g, H.native_gate(g)) for g in "xyzsth"]
    out += [("rz", H.native_gate("rz", -1.3)), ("depol", H.depolarising(0.07)),
            ("ampdamp", H.amplitude_damping(0.2)), ("haar1", H.make_generic("haar1", HS.haar(1, 5))),
            ("kraus1", H.make_generic("kraus1", _kraus(1, 3, 6))),
            ("cnot", H.native_gate("cnot")), ("swap", H.native_gate("swap")),
            ("haar2", H.make_generic("haar2", HS.haar(2, 7))), ("kraus2", H.make_generic("kraus2", _kraus(2, 5, 8))),
            ("toffoli", H.native_gate("toffoli")), ("haar3", H.make_generic("haar3", HS.haar(3, 9))),
            ("kraus3", H.make_generic("kraus3", _kraus(3, 3, 10)))]
    return out


def _pairs(H, HS, n, m, seed):
    rho, obs = H.TiledHermitian(n, m), H.TiledHermitian(n, m)
    psi = HS.rank_psi(n, seed, 4)
    strings = HS.pauli_strings(n, 64, seed + 1)
    return rho, obs, psi, strings


def _duality(H, rho, obs, psi, strings, spec, tg):
    rho.fill_mixture(psi)
    obs.fill_pauli_sum(*strings)
    H.apply(rho, spec, list(tg))
    lhs = H.expectation(rho, obs)
    rho.fill_mixture(psi)
    H.apply(obs, H.dual_channel(spec), list(tg))
    rhs = H.expectation(rho, obs)
    return lhs, rhs, TOL * H.frobenius(rho) * H.frobenius(obs)


@pytest.mark.parametrize("n,m", [(9, 5), (7, 2), (6, 0)])
def test_duality_every_channel(H, HS, n, m):
    rng = np.random.default_rng(40 + n)
    rho, obs, psi, strings = _pairs(H, HS, n, m, 31)
    for name, spec in _channels(H, HS):
        all_t = list(itertools.permutations(range(n), spec.k))
        for i in rng.choice(len(all_t), size=min(6, len(all_t)), replace=False):
            lhs, rhs, bound = _duality(H, rho, obs, psi, strings, spec, all_t[i])
            assert abs(lhs - rhs) <= max(bound, 1e-15), f"{name} {all_t[i]} n={n} m={m}: {lhs} vs {rhs}"
    rho.free()
    obs.free()


@pytest.mark.slow
def test_duality_at_config_size(H, HS):
    """n = 16 (34.4 GB per operator): every regime of the k = 1 / 2 / 3 paths, no CPU result needed."""
    n, m = 16, 5
    rho, obs, psi, strings = _pairs(H, HS, n, m, 33)
    cases = [(H.depolarising(0.01), (3,)), (H.amplitude_damping(0.05), (12,)),
             (H.make_generic("kraus2", _kraus(2, 16, 3)), (2, 9)), (H.make_generic("kraus2", _kraus(2, 4, 4)), (14, 7)),
             (H.make_generic("haar3", HS.haar(3, 5)), (15, 1, 8)), (H.make_generic("kraus3", _kraus(3, 4, 6)), (6, 11, 13)),
             (H.native_gate("cnot"), (0, 15))]
    for spec, tg in cases:
        lhs, rhs, bound = _duality(H, rho, obs, psi, strings, spec, tg)
        print(f"DUALITY n={n} {spec.name} {tg}: {lhs:.15e} vs {rhs:.15e} (bound {bound:.2e})", flush=True)
        assert abs(lhs - rhs) <= bound, f"{spec.name} {tg}: {lhs} vs {rhs}"
    rho.free()
    obs.free()


def _diag_tiles_hermitian(st, n, m):
    """max |T - T^dagger| over the stored diagonal tiles (both halves are stored)."""
    M = 1 << m
    G = max(1, (1 << n) >> m)
    worst = 0.0
    for t in range(G):
        tile = st.download_range((t * (t + 1) // 2 + t) * M * M, M * M).reshape(M, M)
        worst = max(worst, float(np.abs(tile - tile.conj().T).max()))
    return worst


@pytest.mark.parametrize("n,m,nops", [(10, 5, 400), (8, 2, 300), (14, 5, 120)])
def test_trace_and_hermiticity_drift(H, HS, n, m, nops):
    rng = np.random.default_rng(7 * n + m)
    st = H.TiledHermitian(n, m)
    st.fill_mixture(HS.rank_psi(n, 51, 4))
    chans = _channels(H, HS)
    for _ in range(nops):
        name, spec = chans[rng.integers(len(chans))]
        tg = rng.choice(n, size=spec.k, replace=False)
        H.apply(st, spec, [int(t) for t in tg])
    tr = H.trace(st)
    herm = _diag_tiles_hermitian(st, n, m)
    print(f"DRIFT n={n} m={m} ops={nops}: |tr - 1| = {abs(tr - 1.0):.2e}, diagonal-tile hermiticity {herm:.2e}", flush=True)
    assert abs(tr - 1.0) <= 1e-12
    assert herm <= 1e-14
    st.free()


@pytest.mark.parametrize("n,m", [(10, 5), (7, 3)])
def test_linearity(H, HS, n, m):
    a, b = 0.37, -1.9
    x = HS.rho_payload(n, HS.rank_psi(n, 61, 4), m)
    y = HS.pauli_payload(n, HS.pauli_strings(n, 32, 62), m)
    st = H.TiledHermitian(n, m)
    rng = np.random.default_rng(63)
    for name, spec in _channels(H, HS):
        tg = [int(t) for t in rng.choice(n, size=spec.k, replace=False)]
        outs = []
        for payload in (x, y, a * x + b * y):
            st.upload(payload)
            H.apply(st, spec, tg)
            outs.append(st.download())
        scale = np.sqrt(float(np.vdot(outs[2], outs[2]).real)) * 2
        err = float(np.abs(outs[2] - (a * outs[0] + b * outs[1])).max())
        assert err <= TOL * scale, f"{name} {tg}: {err}"
    st.free()


def test_repeat_is_bit_identical(H, HS):
    n, m = 12, 5
    rng = np.random.default_rng(71)
    chans = _channels(H, HS)
    seq = []
    for _ in range(60):
        name, spec = chans[rng.integers(len(chans))]
        seq.append((spec, [int(t) for t in rng.choice(n, size=spec.k, replace=False)]))
    st = H.TiledHermitian(n, m)
    outs = []
    for _ in range(2):
        st.fill_mixture(HS.rank_psi(n, 72, 4))
        for spec, tg in seq:
            H.apply(st, spec, tg)
        outs.append(st.download())
    assert np.array_equal(outs[0].view(np.uint64), outs[1].view(np.uint64))
    st.free()
