"""GPU parity: the B200 engine (through the reference-shaped API, C facade -> C++ host -> C-ABI
-> CUDA) against the CPU oracle (oracle/orkan_oracle.c, itself pinned to the compiled reference
in test_oracle_cpu.py) on identical seeded inputs.

Bar (BASELINE.json north_star): max elementwise |delta| <= 1e-12 * ||X_cpu||_F over
the stored triangle; permutation paths (X, CNOT, SWAP, Toffoli) bit-exact.  Kernel paths and
subcase counters must agree with the reference's ApplyPlan (k = 3 excepted: the reference runs a
dense round trip, this engine runs the tiled regime directly).
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


def _haar(HS, k, seed):
    return HS.haar(k, seed)


def _random_kraus(k, r, seed):
    """Random CPTP Kraus set: blocks of a Haar isometry."""
    rng = np.random.default_rng(seed)
    d = 1 << k
    z = (rng.normal(size=(r * d, d)) + 1j * rng.normal(size=(r * d, d))) / np.sqrt(2)
    q, _ = np.linalg.qr(z)
    return np.stack([q[a * d:(a + 1) * d, :] for a in range(r)])


def _channels(H, HS, oracle):
    """(name, gpu spec, oracle channel) for the library of SPEC.md + config channels."""
    out = []
    for g in "xyzsth":
        out.append((g, H.native_gate(g), oracle.native_gate(g)))
    out.append(("rz", H.native_gate("rz", 0.7), oracle.native_gate("rz", 0.7)))
    out.append(("depol", H.depolarising(0.1), oracle.depolarising(0.1)))
    out.append(("ampdamp", H.amplitude_damping(0.05), oracle.amplitude_damping(0.05)))
    u1 = _haar(HS, 1, 11)
    out.append(("haar1", H.make_generic("haar1", u1), oracle.generic(u1)))
    for g in ("cnot", "swap"):
        out.append((g, H.native_gate(g), oracle.native_gate(g)))
    u2 = _haar(HS, 2, 12)
    out.append(("haar2", H.make_generic("haar2", u2), oracle.generic(u2)))
    k2 = _random_kraus(2, 3, 13)
    out.append(("kraus2", H.make_generic("kraus2", k2), oracle.generic(k2)))
    out.append(("toffoli", H.native_gate("toffoli"), oracle.native_gate("toffoli")))
    u3 = _haar(HS, 3, 14)
    out.append(("haar3", H.make_generic("haar3", u3), oracle.generic(u3)))
    k3 = _random_kraus(3, 2, 15)
    out.append(("kraus3", H.make_generic("kraus3", k3), oracle.generic(k3)))
    return out


def _targets(n, k, limit, rng):
    all_t = list(itertools.permutations(range(n), k))
    if len(all_t) <= limit:
        return all_t
    idx = rng.choice(len(all_t), size=limit, replace=False)
    return [all_t[i] for i in sorted(idx)]


@pytest.mark.parametrize("n,m", [(6, 5), (7, 5), (8, 5), (9, 5), (7, 2), (8, 3), (6, 0), (5, 1), (3, 5), (2, 5),
                                 (10, 4)])
def test_library_parity(H, HS, oracle, orc, n, m):
    if m > n + 2:
        pytest.skip("invalid tile exponent")
    rng = np.random.default_rng(1000 * n + m)
    psi = HS.rank_psi(n, 77 + n, 4)
    base = HS.rho_payload(n, psi, m)
    fro = orc.frobenius(base, n, m)
    st = H.TiledHermitian(n, m)
    for name, spec, och in _channels(H, HS, oracle):
        k = spec.k
        if k > n:
            continue
        limit = {1: 64, 2: 40, 3: 12}[k]
        for tg in _targets(n, k, limit, rng):
            want = base.copy()
            opath, osub = orc.apply(want, n, m, och, list(tg))
            st.upload(base)
            plan = H.apply(st, spec, list(tg))
            got = st.download()
            err = oracle.rel_max_err(got, want, fro)
            exact = name in ("x", "cnot", "swap", "toffoli")
            assert err <= (0.0 if exact else TOL), f"{name} {tg} n={n} m={m}: err {err}"
            if k <= 2:
                assert plan.path == opath, f"{name} {tg}: path {plan.path} vs {opath}"
                assert plan.subcases == osub, f"{name} {tg}: subcases {plan.subcases} vs {osub}"
            else:
                assert plan.path in ("tiled-intra", "tiled-cross", "tiled-mixed", "native-permutation")
    st.free()


# Staging modes of the gather kernel for the FP64 tensor-core transforms (engine.cu plan_gather),
# each hit deterministically at n = 10, m = 5 (units include the diagonal base pairs):
#   k = 3 on one grid bit          -> bulk rows (whole 32 x 32 tiles)
#   k = 3 on two grid bits, in-tile target below bit 3 -> TMA boxes, one quadrant per warp
#   k = 3 on two grid bits, in-tile target at bit 3 / 4 -> TMA boxes, box in the lane constants
#   k = 3 on three grid bits       -> TMA boxes (one per tile)
#   k = 3 on in-tile bits only     -> whole-tile pipeline (scalar two-stage transform)
#   k = 2 on one / two grid bits, or in-tile -> the k = 2 pairing, or promoted to k = 3 (I2 (x) L)
STAGING_CASES = [
    (3, (0, 2, 4)), (3, (4, 1, 3)), (2, (1, 3)), (2, (3, 7)),
    (3, (0, 2, 6)), (3, (6, 4, 1)), (3, (1, 6, 8)), (3, (9, 2, 5)), (3, (0, 7, 9)), (3, (3, 6, 8)),
    (3, (8, 4, 6)), (3, (5, 6, 8)), (3, (9, 7, 5)), (3, (6, 9, 8)), (2, (6, 8)), (2, (9, 5)),
]


@pytest.mark.parametrize("dual", [False, True])
def test_gather_staging_modes(H, HS, oracle, orc, dual):
    n, m = 10, 5
    psi = HS.rank_psi(n, 91, 4)
    base = HS.rho_payload(n, psi, m)
    fro = orc.frobenius(base, n, m)
    st = H.TiledHermitian(n, m)
    for i, (k, tg) in enumerate(STAGING_CASES):
        u = _haar(HS, k, 300 + i)
        spec, och = H.make_generic("u", u), oracle.generic(u)
        if dual:
            spec, och = H.dual_channel(spec), oracle.dual(och)
        want = base.copy()
        orc.apply(want, n, m, och, list(tg))
        st.upload(base)
        H.apply(st, spec, list(tg))
        err = oracle.rel_max_err(st.download(), want, fro)
        assert err <= TOL, f"k={k} {tg} dual={dual}: err {err}"
    st.free()


def _depolarising2(p):
    """Two-qubit depolarising channel: rank 16 (sqrt(1 - p) I, sqrt(p / 15) P for the 15 Paulis)."""
    P = [np.eye(2), np.array([[0, 1], [1, 0]]), np.array([[0, -1j], [1j, 0]]), np.diag([1.0, -1.0])]
    ops = [np.kron(a, b).astype(np.complex128) for a in P for b in P]
    w = [np.sqrt(1 - p)] + [np.sqrt(p / 15)] * 15
    return np.stack([wi * o for wi, o in zip(w, ops)])


@pytest.mark.parametrize("rank", [2, 4, 16])
def test_kraus2_sform_every_pair(H, HS, oracle, orc, rank):
    """k = 2 Kraus sums of rank 2, 4 and 16 (the S-form transform on the FP64 tensor path) on every
    ordered target pair at n = 10, m = 5: in-tile, mixed and cross regimes, diagonal units."""
    n, m = 10, 5
    ops = _depolarising2(0.2) if rank == 16 else _random_kraus(2, rank, 400 + rank)
    spec, och = H.make_generic("k", ops), oracle.generic(ops)
    psi = HS.rank_psi(n, 93, 4)
    base = HS.rho_payload(n, psi, m)
    fro = orc.frobenius(base, n, m)
    st = H.TiledHermitian(n, m)
    worst = 0.0
    for tg in itertools.permutations(range(n), 2):
        want = base.copy()
        orc.apply(want, n, m, och, list(tg))
        st.upload(base)
        H.apply(st, spec, list(tg))
        err = oracle.rel_max_err(st.download(), want, fro)
        worst = max(worst, err)
        assert err <= TOL, f"rank {rank} {tg}: err {err}"
    print(f"kraus2 rank {rank}: worst rel err {worst:.3e} over {n * (n - 1)} pairs")
    st.free()


@pytest.mark.parametrize("rank", [3, 4, 6, 64])
def test_kraus3_sums(H, HS, oracle, orc, rank):
    """k = 3 Kraus sums: rank <= 3 on the direct per-operator DMMA sum, rank >= 4 through the 64 x 64
    transfer matrix (S form on the FP64 tensor path), every regime (in-tile, one / two / three grid
    targets, target orders) at n = 10, m = 5, against the oracle's dense round trip."""
    n, m = 10, 5
    ops = _random_kraus(3, rank, 500 + rank)
    spec, och = H.make_generic("k", ops), oracle.generic(ops)
    psi = HS.rank_psi(n, 95, 4)
    base = HS.rho_payload(n, psi, m)
    fro = orc.frobenius(base, n, m)
    st = H.TiledHermitian(n, m)
    worst = 0.0
    for tg in [(0, 2, 4), (4, 1, 3), (2, 0, 6), (6, 4, 1), (1, 6, 8), (9, 2, 5), (3, 6, 8), (9, 7, 5), (5, 6, 7),
               (8, 9, 7), (0, 9, 1), (7, 3, 9), (4, 9, 6), (8, 4, 6)]:
        want = base.copy()
        orc.apply(want, n, m, och, list(tg))
        st.upload(base)
        H.apply(st, spec, list(tg))
        err = oracle.rel_max_err(st.download(), want, fro)
        worst = max(worst, err)
        assert err <= TOL, f"rank {rank} {tg}: err {err}"
    print(f"kraus3 rank {rank}: worst rel err {worst:.3e}")
    st.free()


@pytest.mark.parametrize("n,m", [(10, 5), (9, 3), (7, 5), (3, 5), (8, 0)])
def test_cx_layer_bit_identical(H, HS, n, m):
    """hs_apply_cx_layer (fusion) equals one native CX after the other, bit for bit: in-tile,
    grid, and mixed pairs in both directions, elements crossing the diagonal, diagonal tiles."""
    rng = np.random.default_rng(100 * n + m)
    psi = HS.rank_psi(n, 19, 4)
    a, b = H.TiledHermitian(n, m), H.TiledHermitian(n, m)
    cx = H.native_gate("cnot")
    for rep in range(4):
        a.fill_mixture(psi)
        b.fill_mixture(psi)
        perm = [int(q) for q in rng.permutation(n)]
        pairs = [(perm[2 * i], perm[2 * i + 1]) for i in range(n // 2)][: 1 + rep * 2]
        for c, t in pairs:
            H.apply(a, cx, [c, t])
        H.apply_cx_layer(b, pairs)
        assert np.array_equal(a.download().view(np.uint64), b.download().view(np.uint64)), (n, m, pairs)
    a.free()
    b.free()


@pytest.mark.parametrize("n,m", [(10, 5), (11, 5), (9, 3), (8, 2)])
def test_cx_layer_sibling_groups_bit_identical(H, HS, n, m):
    """CX layers whose in-tile controls 0 / 1 / 2 have grid targets (cx_layer_kernel takes the sibling
    tiles (ti, tj ^ target bit) together, one or two group bits; groups cut by the diagonal fall back
    to single tiles), mixed with every other pair category, against sequential CX, bit for bit."""
    rng = np.random.default_rng(300 * n + m)
    psi = HS.rank_psi(n, 23, 4)
    a, b = H.TiledHermitian(n, m), H.TiledHermitian(n, m)
    cx = H.native_gate("cnot")
    grid = list(range(m, n))
    for rep in range(6):
        a.fill_mixture(psi)
        b.fill_mixture(psi)
        g = [int(q) for q in rng.permutation(grid)]
        ctl = [[0], [1], [0, 1], [2], [2, 0], [1, 2, 0]][rep]
        pairs = [(c, g[i]) for i, c in enumerate(ctl) if c < m]
        rest = [int(q) for q in rng.permutation([q for q in range(n) if q not in {c for p in pairs for c in p}])]
        pairs += [(rest[2 * i], rest[2 * i + 1]) for i in range(len(rest) // 2)][: rep]
        pairs = [pairs[i] for i in rng.permutation(len(pairs))]
        for c, t in pairs:
            H.apply(a, cx, [c, t])
        H.apply_cx_layer(b, pairs)
        assert np.array_equal(a.download().view(np.uint64), b.download().view(np.uint64)), (n, m, pairs)
    a.free()
    b.free()


def test_generic_path_without_native(H, HS, oracle, orc):
    """allow_native = false routes native gates through the generic engines (kernels.cpp:515)."""
    n, m = 8, 5
    psi = HS.rank_psi(n, 5, 4)
    base = HS.rho_payload(n, psi, m)
    fro = orc.frobenius(base, n, m)
    st = H.TiledHermitian(n, m)
    opts = H.ApplyOptions(allow_native=False)
    for g, k in (("h", 1), ("x", 1), ("y", 1), ("rz", 1), ("cnot", 2), ("swap", 2), ("toffoli", 3)):
        spec, och = H.native_gate(g, 0.3), oracle.native_gate(g, 0.3)
        for tg in [(0,), (4,), (5,), (7,)] if k == 1 else [(7, 2), (1, 6), (5, 6)] if k == 2 else [(7, 0, 5)]:
            want = base.copy()
            orc.apply(want, n, m, och, list(tg), allow_native=False)
            st.upload(base)
            H.apply(st, spec, list(tg), opts)
            assert oracle.rel_max_err(st.download(), want, fro) <= TOL, (g, tg)


def test_device_generators_bit_identical(H, HS):
    for n, m in ((7, 5), (9, 3), (4, 5), (6, 0)):
        psi = HS.rank_psi(n, 3, 4)
        st = H.TiledHermitian(n, m)
        st.fill_mixture(psi)
        assert np.array_equal(st.download().view(np.uint64), HS.rho_payload(n, psi, m).view(np.uint64))
        strings = HS.pauli_strings(n, 64, 99)
        st.fill_pauli_sum(*strings)
        assert np.array_equal(st.download().view(np.uint64), HS.pauli_payload(n, strings, m).view(np.uint64))


def test_expectation_and_trace(H, HS, orc):
    for n, m in ((8, 5), (9, 2), (5, 5)):
        rho = H.TiledHermitian(n, m)
        obs = H.TiledHermitian(n, m)
        psi = HS.rank_psi(n, 21, 4)
        strings = HS.pauli_strings(n, 64, 22)
        rho.fill_mixture(psi)
        obs.fill_pauli_sum(*strings)
        want = orc.expectation(HS.rho_payload(n, psi, m), HS.pauli_payload(n, strings, m), n, m)
        got = H.expectation(rho, obs)
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
        assert abs(H.trace(rho) - 1.0) < 1e-12
        # expectation against the state-vector formula (1/4) sum_i <psi_i|O|psi_i>
        dense_o = orc.to_dense(HS.pauli_payload(n, strings, m), n, m)
        sv = np.mean([np.vdot(p, dense_o @ p).real for p in psi])
        assert abs(got - sv) <= 1e-12 * max(1.0, abs(sv))


def test_errors_match_reference(H):
    st = H.TiledHermitian(4, 2)
    with pytest.raises(IndexError):
        H.apply(st, H.native_gate("h"), [4])
    with pytest.raises(ValueError):
        H.apply(st, H.native_gate("cnot"), [1])
    with pytest.raises(ValueError):
        H.apply(st, H.native_gate("cnot"), [1, 1])
    with pytest.raises(ValueError):
        H.native_gate("nope")
    with pytest.raises(ValueError):
        H.TiledHermitian(0)
    with pytest.raises(ValueError):
        H.TiledHermitian(3, 6)


def test_golden_vectors_gpu(H):
    """The engine reproduces the compiled reference's outputs (tests/golden, make_golden.py)."""
    import json
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    states = {}
    for i, rec in enumerate(meta):
        n, m = rec["n"], rec["m"]
        if (n, m) not in states:
            states[(n, m)] = H.TiledHermitian(n, m)
        st = states[(n, m)]
        st.upload(z[f"in_{n}_{m}"])
        name = rec["name"]
        if rec["kind"] != 0:
            spec = H.native_gate(name, rec["theta"])
        elif name == "depolarising":
            spec = H.depolarising(0.1)
        else:
            spec = H.make_generic(name, z[f"ops_{i}"])
        plan = H.apply(st, spec, rec["targets"])
        want = z[f"out_{i}"]
        fro = float(np.sqrt(np.sum(np.abs(want) ** 2)))  # payload norm >= logical/sqrt(2)
        err = float(np.max(np.abs(st.download() - want))) / fro
        exact = name in ("x", "cnot", "swap", "toffoli")
        assert err <= (0.0 if exact else TOL), (i, name, rec["targets"], err)
        if len(rec["targets"]) <= 2:
            assert plan.path == rec["path"] and list(plan.subcases) == rec["subcases"], (i, name, plan)


def test_device_random_hermitian_matches_reference(H, oracle):
    """random_hermitian / basis_projector generated on the device against the compiled reference's
    own generators (storage.cpp:195-239)."""
    ref = oracle.Reference()
    for n, m, seed in ((8, 5, 3), (9, 3, 11), (4, 5, 7), (7, 0, 2)):
        h = ref.random_hermitian(n, seed, m)
        want = ref.view(h).copy()
        ref.free(h)
        st = H.TiledHermitian(n, m)
        st.fill_random_hermitian(seed)
        got = st.download()
        assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want)), (n, m)
        st.fill_basis_projector(5)
        p = st.download()
        assert p.sum() == 1.0 and np.count_nonzero(p) == 1
