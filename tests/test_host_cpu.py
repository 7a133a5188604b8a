"""CPU tests of the product's host side (no GPU needed): the C-ABI library loads and exports every
entry point declared in include/*.h; the C++ host layer's channel model (through the C facade)
matches the oracle restatement of channel.cpp; the seeded input harness has the properties
BASELINE.json's configs require; bench.py's reference arm honours the JSON contract."""
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b((?:hs|hb)_[a-z0-9_]+)\s*\(", txt)))


@pytest.mark.parametrize("header", ["hs_cuda.h", "hermsim_b200_c.h"])
def test_library_exports_every_declared_symbol(header):
    from paper_2604_15765_b200 import _native
    names = _declared(header)
    assert len(names) > 10
    lib = _native.engine()  # loads without a GPU
    out = subprocess.run(["nm", "-D", "--defined-only", _native.ENGINE_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(lib, n)


def test_engine_reports_missing_device_loudly():
    """No CPU fallback: without a GPU the engine refuses (this container has none)."""
    from paper_2604_15765_b200 import hermsim as H
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is visible")
    with pytest.raises(Exception):
        H.TiledHermitian(4, 2)


def test_channel_model_matches_oracle(oracle, orc):
    from paper_2604_15765_b200 import hermsim as H
    for g in ("x", "y", "z", "s", "t", "h", "cnot", "swap", "toffoli"):
        a, b = H.native_gate(g), oracle.native_gate(g)
        assert np.array_equal(a.kraus, b.ops), g
        assert a.kind == ["generic_kraus", "pauli_x", "pauli_y", "diagonal_phase", "hadamard", "permutation"][b.kind]
        assert np.allclose(a.transfer, orc.transfer_from_kraus(b.ops), atol=1e-15)
    a, b = H.native_gate("rz", 0.7), oracle.native_gate("rz", 0.7)
    assert np.allclose(a.phases, b.phases, atol=1e-16)
    a, b = H.depolarising(0.1), oracle.depolarising(0.1)
    assert np.allclose(a.kraus, b.ops, atol=1e-16)
    # transfer matrix of X is X (x) X; S.vec(|0><0|) = vec(diag(14/15, 1/15))
    x = np.array([[0, 1], [1, 0]])
    assert np.array_equal(H.native_gate("x").transfer, np.kron(x, x))
    v = H.depolarising(0.1).transfer @ np.array([1, 0, 0, 0])
    assert np.allclose(v, [14 / 15, 0, 0, 1 / 15], atol=1e-15)


def test_bind_channel_semantics():
    """bind_channel: first-listed target is the MSB; bound ops re-indexed to ascending qubits."""
    from paper_2604_15765_b200 import hermsim as H
    q, ops, perm = H.bind_channel(H.native_gate("cnot"), [1, 4])  # control 1 < target 4
    assert list(q) == [1, 4]
    assert list(perm) == [0, 3, 2, 1]  # control is now the LOW local bit
    q, ops, perm = H.bind_channel(H.native_gate("cnot"), [4, 1])
    assert list(perm) == [0, 1, 3, 2]
    rng = np.random.default_rng(0)
    u = rng.normal(size=(8, 8)) + 1j * rng.normal(size=(8, 8))
    q, ops, _ = H.bind_channel(H.make_generic("u", u), [5, 0, 3])
    assert list(q) == [0, 3, 5]
    # canonical local bit of listed target j is k-1-j: 5 -> bit 2, 0 -> bit 1, 3 -> bit 0
    def canon(x):  # bound index (bit l <-> sorted[l]) -> canonical index
        b0, b1, b2 = x & 1, (x >> 1) & 1, (x >> 2) & 1  # qubits 0, 3, 5
        return (b2 << 2) | (b0 << 1) | b1
    for r in range(8):
        for c in range(8):
            assert ops[0][r, c] == u[canon(r), canon(c)]


def test_validate_cptni_and_errors():
    from paper_2604_15765_b200 import hermsim as H
    assert H.validate_cptni(H.depolarising(0.1))[0] == "trace_preserving"
    assert H.validate_cptni(H.make_generic("g", [np.sqrt(0.5) * np.eye(2)]))[0] == "trace_non_increasing"
    assert H.validate_cptni(H.make_generic("g", [np.sqrt(2.0) * np.eye(2)]))[0] == "invalid"
    with pytest.raises(ValueError):
        H.make_generic("g", [np.sqrt(2.0) * np.eye(2)], validate=True)
    with pytest.raises(ValueError):
        H.native_gate("nope")
    with pytest.raises(ValueError):
        H.depolarising(1.5)
    with pytest.raises(ValueError):
        H.bind_channel(H.native_gate("cnot"), [2, 2])
    with pytest.raises(ValueError):
        H.make_generic("g", np.zeros((17, 2, 2)))  # rank > 4^k
    # Jacobi eigenvalues of the C++ host layer agree with numpy on a random hermitian
    rng = np.random.default_rng(3)
    a = rng.normal(size=(8, 8)) + 1j * rng.normal(size=(8, 8))
    a = (a + a.conj().T) / 2
    ops = np.linalg.cholesky(np.eye(8) * 50 - a)  # I - sum L^dag L has eigenvalues 1 - eig(50 - a)
    _, _, min_eig = H.validate_cptni(H.make_generic("g", [ops.conj().T]))
    want = np.min(1 - np.linalg.eigvalsh(ops @ ops.conj().T))
    assert abs(min_eig - want) < 1e-9


def test_harness_inputs():
    from paper_2604_15765_b200 import harness as HS
    n = 6
    psi = HS.rank_psi(n, 11, 4)
    assert np.allclose(np.linalg.norm(psi, axis=1), 1.0, atol=1e-14)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    orc = O.Oracle()
    rho = orc.to_dense(HS.rho_payload(n, psi), n, 5)
    want = sum(np.outer(p, p.conj()) for p in psi) / 4
    assert np.allclose(rho, want, atol=1e-15)
    assert abs(np.trace(rho).real - 1) < 1e-14 and np.linalg.matrix_rank(rho, tol=1e-10) == 4
    strings = HS.pauli_strings(n, 64, 5)
    o = orc.to_dense(HS.pauli_payload(n, strings), n, 5)
    assert np.allclose(o, o.conj().T)
    # Pauli-sum payload against explicit Kronecker products
    P = {0: np.eye(2), 1: np.array([[0, 1], [1, 0]]), 2: np.array([[0, -1j], [1j, 0]]), 3: np.diag([1, -1])}
    x, z, ny, coef = strings
    ref_o = np.zeros((1 << n, 1 << n), np.complex128)
    for s in range(64):
        m = np.ones((1, 1))
        for q in reversed(range(n)):
            xb, zb = (int(x[s]) >> q) & 1, (int(z[s]) >> q) & 1
            m = np.kron(m, P[{(0, 0): 0, (1, 0): 1, (1, 1): 2, (0, 1): 3}[(xb, zb)]])
        ref_o += coef[s] * m
    assert np.allclose(o, ref_o, atol=1e-13)
    u = HS.haar(3, 9)
    assert np.allclose(u @ u.conj().T, np.eye(8), atol=1e-14)
    assert HS.haar(2, 4).shape == (4, 4)


def test_config_op_sequences():
    from paper_2604_15765_b200 import harness as HS
    assert len(HS.config_ops("c0")) == 12
    assert len(HS.config_ops("c1")) == 364
    assert len(HS.config_ops("c2")) == 32
    c3 = HS.config_ops("c3")
    assert len(c3) == 100
    for layer in range(20):
        qs = [q for op in c3[5 * layer: 5 * layer + 5] for q in op.targets]
        assert len(set(qs)) == 15  # disjoint triples, one idle qubit
    c4 = HS.config_ops("c4")
    assert len(c4) == 590
    for layer in range(10):
        cx = [op for op in c4[59 * layer: 59 * layer + 59] if op.kind == "cnot"]
        qs = [q for op in cx for q in op.targets]
        assert len(cx) == 8 and len(set(qs)) == 16 and {14, 15, 16} <= set(qs)
        thetas = [op.param for op in c4[59 * layer: 59 * layer + 34] if op.kind == "rz"]
        assert len(thetas) == 17 and all(0 <= t < 2 * np.pi for t in thetas)


def test_bench_reference_arm_contract():
    """bench.py --impl reference prints one JSON line with the contract's keys (small n)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "9",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_fusion_plan_counts():
    """Fusion planner (host only): C2 at n = 16 -> one in-tile program + one pass per grid qubit;
    C4's Rz/H run -> one program + one pass per grid qubit; k >= 2 ops end a run."""
    from paper_2604_15765_b200 import fusion
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    dep, amp = H.depolarising(0.01), H.amplitude_damping(0.05)
    ops = [(dep if op.kind == "depol" else amp, list(op.targets)) for op in HS.config_ops("c2", 16)]
    plan = fusion.plan_sequence(ops, 16, 5, grid_groups=1)
    assert plan.ops == 32 and plan.launches == 12
    assert plan.items[0][0] == "program" and [s.qubit for s in plan.items[0][1]] == [0, 1, 2, 3, 4]
    assert [fusion._kind(s) for s in plan.items[0][1]] == [3] * 5  # depolarising o amplitude damping
    assert all(it[0] == "step" and it[1].count == 2 for it in plan.items[1:])
    h, cx = H.native_gate("h"), H.native_gate("cnot")
    seq = [(H.native_gate("rz", 0.3), [q]) for q in range(8)] + [(h, [q]) for q in range(8)] + [(cx, [7, 1])] + [(h, [6])]
    plan = fusion.plan_sequence(seq, 8, 5, pair_unitaries=False, grid_groups=1)
    kinds = [it[0] for it in plan.items]
    assert kinds == ["program", "step", "step", "step", "op", "step"]
    grouped = fusion.plan_sequence(ops, 16, 5)  # C2: grid qubits three at a time
    assert [it[0] for it in grouped.items] == ["program"] + ["gprogram"] * 3 + ["gprogram"]
    assert [len(it[1]) for it in grouped.items[1:]] == [3, 3, 3, 2]
    paired = fusion.plan_sequence(seq, 8, 5, grid_groups=1)  # grid qubits 5, 6 share a pass as H Rz (x) H Rz
    assert [it[0] for it in paired.items] == ["program", "op", "step", "op", "step"]
    assert paired.items[1][2] == [5, 6] and paired.items[1][1].k == 2
    assert paired.items[2][1].qubit == 7 and paired.items[-1][1].lone_h
    assert plan.items[-1][1].lone_h
    # Rz then H: a chain of two cheap steps per qubit (diagonal, Hadamard) rather than one general
    # transfer -- a qubit's chain shares one shared-memory round trip, so only arithmetic counts
    assert [fusion._kind(s) for s in plan.items[0][1]] == [2, 1] * 5
    assert [s.qubit for s in plan.items[0][1]] == [0, 0, 1, 1, 2, 2, 3, 3, 4, 4]
    # C1: CX then Haar U on each ordered pair -> one composed unitary per pair, U @ CX in the pair's order
    c1 = [(cx if op.kind == "cnot" else H.make_generic("haar", op.matrix), list(op.targets))
          for op in HS.config_ops("c1", 14)]
    p1 = fusion.plan_sequence(c1, 14, 5)
    assert p1.ops == 364 and p1.launches == 182
    assert np.allclose(p1.items[0][1].kraus[0], c1[1][0].kraus[0] @ cx.kraus[0]) and p1.items[0][2] == c1[0][1]
    # a reordered pair: U written for [b, a] is re-indexed to [a, b] first
    u = HS.haar(2, 9)
    p2 = fusion.plan_sequence([(cx, [6, 2]), (H.make_generic("u", u), [2, 6])], 8, 5)
    assert p2.launches == 1
    assert np.allclose(p2.items[0][1].kraus[0], fusion.reorder_targets(u, [2, 6], [6, 2]) @ cx.kraus[0])
    assert np.allclose(fusion.reorder_targets(cx.kraus[0], [0, 1], [1, 0]),
                       np.array([[1, 0, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0], [0, 1, 0, 0]]))
    # C4: the CX of each layer's matching run as one CX layer (disjoint pairs)
    c4 = []
    for op in HS.config_ops("c4", 17):
        if op.kind == "rz":
            c4.append((H.native_gate("rz", op.param), list(op.targets)))
        elif op.kind == "h":
            c4.append((h, list(op.targets)))
        elif op.kind == "cnot":
            c4.append((cx, list(op.targets)))
        else:
            c4.append((H.depolarising(op.param), list(op.targets)))
    p4 = fusion.plan_sequence(c4, 17, 5)
    layers = [it for it in p4.items if it[0] == "cxlayer"]
    assert p4.ops == 590 and len(layers) == 10 and all(len(it[1]) == 8 for it in layers)
    assert p4.launches == 65
    # CX sharing a qubit end a layer; a lone CX stays a plain operation
    p5 = fusion.plan_sequence([(cx, [0, 1]), (cx, [2, 3]), (cx, [1, 4]), (h, [0])], 8, 5)
    assert [it[0] for it in p5.items] == ["cxlayer", "op", "program"]
    # composition order: S(second) @ S(first)
    s_rz = fusion.transfer_rowstacked(H.native_gate("rz", 0.3).kraus)
    s_h = fusion.transfer_rowstacked(h.kraus)
    assert np.allclose(plan.items[1][1].s, s_h @ s_rz)


def test_reorder_targets_properties():
    """fusion.reorder_targets: the same operator listed in another target order (first listed =
    most significant bit): kron factors swap places, and reordering back is the identity."""
    from paper_2604_15765_b200 import fusion
    rng = np.random.default_rng(5)
    a, b, c = (rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2)) for _ in range(3))
    u = np.kron(np.kron(a, b), c)  # targets [7, 2, 4]
    assert np.allclose(fusion.reorder_targets(u, [7, 2, 4], [4, 7, 2]), np.kron(np.kron(c, a), b))
    assert np.allclose(fusion.reorder_targets(u, [7, 2, 4], [2, 4, 7]), np.kron(np.kron(b, c), a))
    v = rng.normal(size=(8, 8)) + 1j * rng.normal(size=(8, 8))
    w = fusion.reorder_targets(fusion.reorder_targets(v, [0, 1, 2], [2, 0, 1]), [2, 0, 1], [0, 1, 2])
    assert np.allclose(w, v)


def test_ohrm_header_validation_without_device(tmp_path):
    """hs_state_load validates the OHRM header (storage_io.cpp:58-83) before touching a device:
    each malformed header fails with the reference's IoErrorKind."""
    from paper_2604_15765_b200 import _native as nat
    from paper_2604_15765_b200 import hermsim as H

    def hdr(magic=b"OHRM", ver=1, tag=2, n=6, m=3):
        return magic + ver.to_bytes(4, "little") + bytes([tag, n, m, 0, 0, 0, 0, 0])

    cases = [(hdr(magic=b"OHRX"), "bad_magic"), (hdr(ver=2), "bad_version"), (hdr(tag=3), "bad_header"),
             (hdr(n=0), "bad_header"), (hdr(n=31), "bad_header"), (hdr(m=9), "bad_header"),
             (hdr(tag=0, m=1), "bad_header"), (b"OHRM\x01\x00", "truncated")]
    for i, (data, kind) in enumerate(cases):
        p = tmp_path / f"h{i}.ohrm"
        p.write_bytes(data)
        with pytest.raises(nat.IoError) as ei:
            H.TiledHermitian.load(str(p))
        assert ei.value.kind == kind, (data, str(ei.value))
    with pytest.raises(nat.IoError) as ei:
        H.TiledHermitian.load(str(tmp_path / "missing.ohrm"))
    assert ei.value.kind == "io_failure"
    p = tmp_path / "dense.ohrm"
    p.write_bytes(hdr(tag=0, m=0))
    with pytest.raises(NotImplementedError):  # dense / packed are not device formats
        H.TiledHermitian.load(str(p))
