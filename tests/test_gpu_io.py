"""OHRM save / load (storage_io.cpp:34-118) between HBM and files, against the compiled reference's
own save / load: byte-identical payloads both ways; truncation and trailing bytes rejected."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m", [(7, 3), (10, 5), (4, 5)])
def test_roundtrip_with_reference(tmp_path, oracle, n, m):
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    ref = oracle.Reference()
    st = H.TiledHermitian(n, m)
    st.fill_mixture(HS.rank_psi(n, 5, 4))
    H.apply(st, H.depolarising(0.2), [min(n - 1, 6)])
    p1 = str(tmp_path / "gpu.ohrm")
    st.save(p1)
    h = ref.load(p1)  # the reference reads our file
    assert np.array_equal(ref.view(h).view(np.uint64), st.download().view(np.uint64))
    H_ = ref.random_hermitian(n, 99, m)
    p2 = str(tmp_path / "ref.ohrm")
    ref.save(H_, p2)
    back = H.TiledHermitian.load(p2)  # we read the reference's file
    assert np.array_equal(back.download().view(np.uint64), ref.view(H_).view(np.uint64))
    assert os.path.getsize(p1) == 16 + st.element_count() * 16
    ref.free(h)
    ref.free(H_)


def test_truncated_and_trailing(tmp_path):
    from paper_2604_15765_b200 import _native as nat
    from paper_2604_15765_b200 import hermsim as H
    st = H.TiledHermitian(8, 5)
    st.fill_mixture(np.eye(4, 1 << 8, dtype=np.complex128))
    p = tmp_path / "a.ohrm"
    st.save(str(p))
    data = p.read_bytes()
    (tmp_path / "t.ohrm").write_bytes(data[:-16])
    (tmp_path / "x.ohrm").write_bytes(data + b"\0")
    with pytest.raises(nat.IoError) as e1:
        H.TiledHermitian.load(str(tmp_path / "t.ohrm"))
    with pytest.raises(nat.IoError) as e2:
        H.TiledHermitian.load(str(tmp_path / "x.ohrm"))
    assert e1.value.kind == "truncated" and e2.value.kind == "length_mismatch"
