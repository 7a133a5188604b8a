"""Sharded engine (XOR blocks) against the single-GPU engine: P shards driven from one process on one
B200 (exchange by device copies, kernels launched one after another -- no kernel waits on another).
The same per-element arithmetic runs either way, so the results must be bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ops(H, HS, n):
    u2, u3 = HS.haar(2, 5), HS.haar(3, 6)
    top = n - 1
    return [
        (H.native_gate("h"), [0]), (H.native_gate("h"), [top]), (H.depolarising(0.01), [top - 1]),
        (H.amplitude_damping(0.05), [top]), (H.native_gate("rz", 0.37), [top]), (H.native_gate("rz", 1.1), [2]),
        (H.native_gate("cnot"), [top, 3]), (H.native_gate("cnot"), [1, top - 2]), (H.native_gate("cnot"), [6, 7]),
        (H.make_generic("u2", u2), [top, 5]), (H.make_generic("u2", u2), [2, top - 1]),
        (H.make_generic("u3", u3), [top, 4, 0]), (H.make_generic("u3", u3), [6, 5, 8]),
        (H.native_gate("y"), [top]), (H.native_gate("swap"), [top - 2, 1]), (H.depolarising(0.02), [5]),
    ]


@pytest.mark.parametrize("n,P", [(9, 2), (10, 4), (11, 8), (10, 2)])
def test_sharded_bit_identical(n, P):
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import ShardGroup
    psi = HS.rank_psi(n, 42, 4)
    ref = H.TiledHermitian(n)
    ref.fill_mixture(psi)
    grp = ShardGroup(n, 5, P)
    grp.fill_mixture(psi)
    assert np.array_equal(grp.download_full().view(np.uint64), ref.download().view(np.uint64))
    opts = H.ApplyOptions(count_subcases=False)
    for spec, tg in _ops(H, HS, n):
        if len([q for q in tg if q >= grp.layout.top0]) > 1:
            continue
        H.apply(ref, spec, tg, opts)
        grp.apply(spec, tg)
        got, want = grp.download_full(), ref.download()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (spec.name, tg, np.max(np.abs(got - want)))
    assert abs(grp.trace() - H.trace(ref)) < 1e-13
    obs = ShardGroup(n, 5, P)
    obs_ref = H.TiledHermitian(n)
    strings = HS.pauli_strings(n, 16, 3)
    obs.fill_pauli_sum(*strings)
    obs_ref.fill_pauli_sum(*strings)
    assert abs(grp.expectation(obs) - H.expectation(ref, obs_ref)) < 1e-13


def test_two_top_targets_refused():
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import ShardGroup
    grp = ShardGroup(10, 5, 4)
    with pytest.raises(NotImplementedError):
        grp.apply(H.native_gate("cnot"), [9, 8])
