"""Format conversions on the device against the compiled reference's own
hermsim::to_dense / convert (/root/reference/proj/src/storage.cpp:241-292), bit-exact.

Inputs are arbitrary payloads (not hermitian): the conversions are defined element by element, so a
payload whose diagonal tiles' halves disagree pins the reference's "diagonal tile holds both halves"
rule (storage.cpp:271-273) and fill_from_lower's mirror rule (storage.cpp:170-186) exactly.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [(1, 0), (1, 3), (2, 2), (3, 5), (5, 5), (6, 1), (7, 3), (8, 5), (9, 4), (10, 5)]


@pytest.fixture(scope="module")
def H():
    from paper_2604_15765_b200 import hermsim
    if hermsim.device_count() < 1:
        pytest.fail("no CUDA device visible")
    return hermsim


def _noise(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.normal(size=shape) + 1j * rng.normal(size=shape)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("n,m", CASES)
def test_to_dense_and_packed_bit_exact(H, ref, n, m):
    h = ref.create(n, m)
    payload = _noise(ref.view(h).shape, 100 * n + m)
    ref.view(h)[:] = payload
    st = H.TiledHermitian(n, m)
    st.upload(payload)
    d = ref.convert(h, "dense")
    p = ref.convert(h, "packed")
    want_d, want_p = ref.view(d).reshape(1 << n, 1 << n), ref.view(p)
    assert np.array_equal(_bits(st.to_dense()), _bits(want_d))
    assert np.array_equal(_bits(st.to_packed()), _bits(want_p))
    for x in (h, d, p):
        ref.free(x)
    st.free()


@pytest.mark.parametrize("n,m", CASES)
def test_from_dense_and_packed_bit_exact(H, ref, n, m):
    N = 1 << n
    dense = _noise((N, N), 7 * n + m)
    hd = ref.create_dense(n, dense)
    ht = ref.convert(hd, "tiled", m)
    hp = ref.convert(hd, "packed")
    htp = ref.convert(hp, "tiled", m)
    st = H.TiledHermitian(n, m)
    st.from_dense(dense)
    assert np.array_equal(_bits(st.download()), _bits(ref.view(ht)))
    st.zero()
    st.from_packed(ref.view(hp).copy())
    assert np.array_equal(_bits(st.download()), _bits(ref.view(htp)))
    for x in (hd, ht, hp, htp):
        ref.free(x)
    st.free()


@pytest.mark.parametrize("n,m1,m2", [(3, 5, 0), (4, 2, 5), (7, 5, 3), (9, 1, 5), (10, 5, 4), (10, 3, 3)])
def test_retile_bit_exact(H, ref, n, m1, m2):
    h = ref.create(n, m1)
    payload = _noise(ref.view(h).shape, 31 * n + m1 + m2)
    ref.view(h)[:] = payload
    want = ref.convert(h, "tiled", m2)
    src = H.TiledHermitian(n, m1)
    src.upload(payload)
    dst = H.convert(src, "tiled", m2)
    assert dst.tile_exp() == m2
    assert np.array_equal(_bits(dst.download()), _bits(ref.view(want)))
    for x in (h, want):
        ref.free(x)
    src.free()
    dst.free()


def test_conversions_on_device_buffers_and_bands(H, ref):
    """n = 13: the dense matrix (1.07 GB) crosses several 256 MB staging bands on the host path; the
    device path writes a cudaMalloc'd buffer; both equal the reference; dense -> tiled -> dense round
    trip of a hermitian operator is the identity."""
    from paper_2604_15765_b200 import _native as nat
    n, m = 13, 5
    N = 1 << n
    L = nat.engine()
    st = H.TiledHermitian(n, m)
    h = ref.random_hermitian(n, 11, m)
    st.upload(ref.view(h).copy())
    d = ref.convert(h, "dense")
    want = ref.view(d).reshape(N, N)
    got = st.to_dense()
    assert np.array_equal(_bits(got), _bits(want))
    buf = ctypes.c_void_p()
    nat.check(L.hs_device_alloc(0, N * N * 16, ctypes.byref(buf)))
    nat.check(L.hs_state_to_dense(st.handle, buf, 1))
    st.synchronize()
    dev = np.empty((N, N), np.complex128)
    nat.check(L.hs_copy_d2h(0, dev.ctypes.data, buf, N * N * 16))
    assert np.array_equal(_bits(dev), _bits(want))
    st2 = H.TiledHermitian(n, m)
    nat.check(L.hs_state_from_dense(st2.handle, buf, 1))
    assert np.array_equal(_bits(st2.download()), _bits(st.download()))
    nat.check(L.hs_device_free(0, buf))
    p = ref.convert(h, "packed")
    assert np.array_equal(_bits(st.to_packed()), _bits(ref.view(p)))
    for x in (h, d, p):
        ref.free(x)
    st.free()
    st2.free()


def test_conversion_refusals(H):
    from paper_2604_15765_b200 import _native as nat
    st = H.TiledHermitian(6, 5)
    with pytest.raises(ValueError):
        st.from_dense(np.zeros((8, 8), np.complex128))
    with pytest.raises(ValueError):
        H.convert(st, "csr")
    other = H.TiledHermitian(7, 5)
    with pytest.raises(ValueError):
        nat.check(nat.engine().hs_state_convert(st.handle, other.handle))
    st.free()
    other.free()
