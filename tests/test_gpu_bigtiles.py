"""Tile exponents m > 5 (the reference accepts m in [0, n + 2], /root/reference/proj/src/storage.cpp:12-20).

The engine keeps such an operator in HBM in the m = 5 layout (every kernel unchanged) and converts
to and from the user's m layout at the boundary (upload / download / save / load / info; the retile
kernel of engine_convert.cuh).  These cases check, against the compiled reference at the same m:
the payload round trip, a sequence of operations of every regime (values at 1e-12 * ||X||_F, the
path tags and subcase counters the reference reports for that m), and OHRM files both ways.
"""
import os

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


def _ops(H, O, HS, n):
    u2, u3 = HS.haar(2, 5), HS.haar(3, 6)
    k3 = HS.random_kraus_ops(3, 4, 9)
    q = [0, n // 2, n - 1]
    return [(H.native_gate("h"), O.native_gate("h"), [q[1]]),
            (H.depolarising(0.1), O.depolarising(0.1), [q[2]]),
            (H.depolarising(0.1), O.depolarising(0.1), [q[0]]),
            (H.native_gate("cnot"), O.native_gate("cnot"), [q[2], q[0]]),
            (H.native_gate("rz", 0.3), O.native_gate("rz", 0.3), [q[1]]),
            (H.make_generic("u2", u2), O.generic(u2), [q[0], q[2]]),
            (H.make_generic("u2", u2), O.generic(u2), [q[1], q[2]]),
            (H.make_generic("u3", u3), O.generic(u3), [q[2], q[0], q[1]]),
            (H.make_generic("k3", k3), O.generic(k3), [q[0], q[1], q[2]])]


@pytest.mark.parametrize("n,m", [(4, 6), (5, 7), (7, 6), (8, 7), (9, 6), (10, 8)])
def test_big_tiles_vs_reference(H, oracle, ref, n, m, tmp_path):
    from paper_2604_15765_b200 import harness as HS
    h = ref.random_hermitian(n, 100 + n, m)
    payload = ref.view(h).copy()
    st = H.TiledHermitian(n, m)
    assert st.tile_exp() == m and st.element_count() == payload.size
    st.upload(payload)
    assert np.array_equal(st.download().view(np.uint64), payload.view(np.uint64))
    orc = oracle.Oracle()
    fro = orc.frobenius(payload, n, m)
    opts = H.ApplyOptions(count_subcases=True)
    for spec, och, tg in _ops(H, oracle, HS, n):
        plan = H.apply(st, spec, tg, opts)
        rpath, rsub = ref.apply(h, och, tg, threads=4)
        if len(tg) < 3:  # k = 3: the reference's dense fallback (this engine runs it tiled)
            assert plan.path == rpath, (tg, plan.path, rpath)
            assert tuple(plan.subcases) == rsub, (tg, plan.subcases, rsub)
        err = oracle.rel_max_err(st.download(), ref.view(h), fro)
        assert err <= TOL, (spec.name, tg, err)
    # OHRM both ways at this m
    p1, p2 = str(tmp_path / "gpu.ohrm"), str(tmp_path / "ref.ohrm")
    st.save(p1)
    h2 = ref.load(p1)
    assert np.array_equal(ref.view(h2).view(np.uint64), st.download().view(np.uint64))
    ref.save(h, p2)
    st2 = H.TiledHermitian.load(p2)
    assert st2.tile_exp() == m
    assert np.array_equal(st2.download().view(np.uint64), ref.view(h).view(np.uint64)) or \
        oracle.rel_max_err(st2.download(), ref.view(h), fro) <= TOL
    for x in (h, h2):
        ref.free(x)
    st.free()
    st2.free()
    _ = os


def test_big_tiles_refuse_sharding(H):
    from paper_2604_15765_b200 import _native as nat
    import ctypes
    out = ctypes.c_void_p()
    rc = nat.engine().hs_state_create_sharded(9, 6, 0, 2, 0, ctypes.byref(out))
    assert rc == -5  # HS_ERR_UNSUPPORTED
