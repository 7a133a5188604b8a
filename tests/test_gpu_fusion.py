"""Fused sequences (paper_2604_15765_b200/fusion.py) against one-op-at-a-time application
on the GPU, and the compiled reference on the same inputs: max |delta| <= 1e-12 * ||X||_F."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _seq(H, HS, name, n):
    if name == "c2":
        return [(H.depolarising(0.01) if op.kind == "depol" else H.amplitude_damping(0.05), list(op.targets))
                for op in HS.config_ops("c2", n)]
    if name == "c0":
        return [(H.native_gate("h"), list(op.targets)) for op in HS.config_ops("c0", n)]
    if name == "c1":  # CX then Haar U4 on ordered pairs: composed per pair, plus a reordered pair
        out = [(H.native_gate("cnot") if op.kind == "cnot" else H.make_generic("haar", op.matrix), list(op.targets))
               for op in HS.config_ops("c1", n)][:60]
        return out + [(H.native_gate("cnot"), [6, 2]), (H.make_generic("haar", HS.haar(2, 9)), [2, 6])]
    out = []
    # two layers (Rz, H, CX matching, depolarising): the second layer's chains start with the first's
    # depolarising composed with Rz (step kind 4)
    for op in HS.config_ops("c4", n)[: 7 * n]:
        if op.kind == "rz":
            out.append((H.native_gate("rz", op.param), list(op.targets)))
        elif op.kind == "h":
            out.append((H.native_gate("h"), list(op.targets)))
        elif op.kind == "cnot":
            out.append((H.native_gate("cnot"), list(op.targets)))
        else:
            out.append((H.depolarising(op.param), list(op.targets)))
    return out


@pytest.mark.parametrize("name,n,m", [("c2", 10, 5), ("c2", 9, 3), ("c0", 9, 5), ("c4", 11, 5), ("c4", 8, 2),
                                      ("c1", 10, 5), ("c1", 8, 3)])
def test_fused_equals_sequential(name, n, m):
    from paper_2604_15765_b200 import fusion
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    psi = HS.rank_psi(n, 11, 4)
    a, b = H.TiledHermitian(n, m), H.TiledHermitian(n, m)
    a.fill_mixture(psi)
    b.fill_mixture(psi)
    ops = _seq(H, HS, name, n)
    opts = H.ApplyOptions(count_subcases=False)
    for spec, tg in ops:
        H.apply(a, spec, tg, opts)
    plan = fusion.apply_sequence(b, ops)
    assert plan.launches < len(ops)
    want, got = a.download(), b.download()
    fro = H.frobenius(a)
    assert np.max(np.abs(got - want)) <= 1e-12 * fro, (name, plan.launches)


@pytest.mark.parametrize("n,seed", [(10, 1), (11, 2), (12, 3)])
def test_fused_random_qubit_subsets(n, seed):
    """Runs of single-qubit operations on random qubit subsets, in random order: programs on 1-5
    in-tile qubits (every pair the shuffle-paired passes can meet, e.g. (1, 4), (0, 3)), grid programs
    on 2 and 3 grid qubits that are not neighbours, every step kind (transfer matrix, Hadamard,
    diagonal, real pair, real pair with complex diagonal, butterfly), against one-op-at-a-time."""
    from paper_2604_15765_b200 import fusion
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    m = 5
    rng = np.random.default_rng(500 + seed)
    makers = [lambda: H.depolarising(float(rng.uniform(0.01, 0.2))), lambda: H.amplitude_damping(float(rng.uniform(0.01, 0.3))),
              lambda: H.native_gate("rz", float(rng.uniform(-3, 3))), lambda: H.native_gate("h"),
              lambda: H.native_gate("s"), lambda: H.make_generic("haar1", HS.haar(1, int(rng.integers(1 << 20))))]
    psi = HS.rank_psi(n, 13, 4)
    a, b = H.TiledHermitian(n, m), H.TiledHermitian(n, m)
    opts = H.ApplyOptions(count_subcases=False)
    for rep in range(8):
        a.fill_mixture(psi)
        b.fill_mixture(psi)
        qs = [int(q) for q in rng.choice(n, size=int(rng.integers(2, n + 1)), replace=False)]
        ops = []
        for _ in range(int(rng.integers(1, 4))):  # up to three operations per qubit, interleaved over the qubits
            for q in rng.permutation(qs):
                ops.append((makers[int(rng.integers(len(makers)))](), [int(q)]))
        for spec, tg in ops:
            H.apply(a, spec, tg, opts)
        plan = fusion.apply_sequence(b, ops)
        want, got = a.download(), b.download()
        fro = H.frobenius(a)
        assert np.max(np.abs(got - want)) <= 1e-12 * fro, (n, rep, sorted(qs), plan.launches)
    a.free()
    b.free()


def test_fused_against_reference(oracle):
    """The fused C2 pass against the compiled reference applying the same 2n operations."""
    from paper_2604_15765_b200 import fusion
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    n, m = 10, 5
    psi = HS.rank_psi(n, 3, 4)
    want = HS.rho_payload(n, psi, m)
    ref = oracle.Reference()
    h = ref.create(n, m, want)
    for op in HS.config_ops("c2", n):
        ch = oracle.depolarising(op.param) if op.kind == "depol" else oracle.amplitude_damping(op.param)
        ref.apply(h, ch, list(op.targets), threads=4)
    want = ref.view(h).copy()
    ref.free(h)
    st = H.TiledHermitian(n, m)
    st.fill_mixture(psi)
    fusion.apply_sequence(st, _seq(H, HS, "c2", n))
    got = st.download()
    assert oracle.rel_max_err(got, want, oracle.Oracle().frobenius(want, n, m)) <= 1e-12
