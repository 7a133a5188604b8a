"""CUDA-graph capture of an operation sequence (hermsim.capture / hs_graph_*): replaying the graph
equals applying the sequence again, bit for bit; uncapturable operations fail loudly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _seq(H, HS, n):
    return [(H.depolarising(0.02), [0]), (H.amplitude_damping(0.1), [n - 1]), (H.native_gate("h"), [6]),
            (H.native_gate("cnot"), [n - 1, 2]), (H.make_generic("u2", HS.haar(2, 1)), [7, n - 2]),
            (H.make_generic("u3", HS.haar(3, 2)), [n - 1, 1, 6]), (H.native_gate("rz", 0.4), [3])]


def test_graph_replay_bit_identical():
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    n = 10
    psi = HS.rank_psi(n, 5, 4)
    a, b = H.TiledHermitian(n), H.TiledHermitian(n)
    a.fill_mixture(psi)
    b.fill_mixture(psi)
    opts = H.ApplyOptions(count_subcases=False)
    seq = _seq(H, HS, n)
    with H.capture(b) as g:  # capture records, does not run
        for spec, tg in seq:
            H.apply(b, spec, tg, opts)
    assert g.nodes() >= len(seq)
    assert np.array_equal(b.download().view(np.uint64), a.download().view(np.uint64))
    for _ in range(3):
        for spec, tg in seq:
            H.apply(a, spec, tg, opts)
        g.launch()
    assert np.array_equal(b.download().view(np.uint64), a.download().view(np.uint64))


def test_graph_refuses_uncapturable():
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    st = H.TiledHermitian(9)
    # k = 3 Kraus sets of rank >= 3 run in the hermitian-basis form, whose real 64 x 64 matrix is built
    # on the host and uploaded the first time a state sees the set: refused inside a capture then ...
    ops = np.stack([np.sqrt(0.2) * HS.haar(3, 3 + i) for i in range(5)])
    k3 = H.make_generic("k3", ops)
    with pytest.raises(Exception):
        with H.capture(st):
            H.apply(st, k3, [8, 2, 0])
    # ... and capturable once the state has it cached (the replay reads the cached device copy)
    psi = HS.rank_psi(9, 6, 4)
    a, b = H.TiledHermitian(9), H.TiledHermitian(9)
    a.fill_mixture(psi)
    b.fill_mixture(psi)
    # the cache holds the BOUND set (bind_channel relabels the local basis by the target order):
    # warm it with a triple of the same order pattern as the captured one (descending)
    H.apply(a, k3, [7, 3, 1])
    H.apply(b, k3, [7, 3, 1])
    with H.capture(a) as g:
        H.apply(a, k3, [8, 2, 0])
    g.launch()
    H.apply(b, k3, [8, 2, 0])
    assert np.array_equal(a.download().view(np.uint64), b.download().view(np.uint64))


def test_graph_of_small_kraus_sum():
    """A k = 3 Kraus sum of 2 operators (tensor-core gather, coefficients in the kernel parameters)
    is capturable and replays bit-identically."""
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    n = 9
    psi = HS.rank_psi(n, 4, 4)
    a, b = H.TiledHermitian(n), H.TiledHermitian(n)
    a.fill_mixture(psi)
    b.fill_mixture(psi)
    k3 = H.make_generic("k3", np.stack([np.sqrt(0.5) * HS.haar(3, 3), np.sqrt(0.5) * HS.haar(3, 4)]))
    with H.capture(a) as g:
        H.apply(a, k3, [8, 2, 0])
    g.launch()
    H.apply(b, k3, [8, 2, 0])
    assert np.array_equal(a.download().view(np.uint64), b.download().view(np.uint64))


def test_graph_of_fused_sequence():
    """A fused C2-style sequence (in-tile program + grid programs) captured and replayed equals the
    fused sequence applied again."""
    from paper_2604_15765_b200 import fusion
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    n = 10
    psi = HS.rank_psi(n, 8, 4)
    a, b = H.TiledHermitian(n), H.TiledHermitian(n)
    a.fill_mixture(psi)
    b.fill_mixture(psi)
    ops = [(H.depolarising(0.01), [q]) for q in range(n)] + [(H.amplitude_damping(0.05), [q]) for q in range(n)]
    plan = fusion.plan_sequence(ops, n, 5)
    with H.capture(b) as g:
        fusion.execute(b, plan)
    for _ in range(2):
        fusion.execute(a, plan)
        g.launch()
    assert np.array_equal(b.download().view(np.uint64), a.download().view(np.uint64))
