"""Seeded synthetic workloads of BASELINE.json's configs.

No public dataset is involved: every config is defined by its shape, so seeded synthetic inputs
stand in.  All randomness comes from the reference's counter-based
``gaussian_entry`` (storage.cpp:22-44) restated in ``csrc/harness.c`` so the GPU arm, the CPU
reference arm and the tests see bit-identical inputs.

An op sequence is a list of ``Op`` records; ``kind`` is one of ``h``, ``rz``, ``cnot``, ``depol``,
``ampdamp``, ``unitary``, ``unitary_dual``, ``kraus`` (a generic Kraus set, ``matrix`` of shape
(rank, 2^k, 2^k)) with constructor-order targets (first = MSB).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat

SEEDS = {"c0": 0xC0FFEE00, "c1": 0xC0FFEE01, "c2": 0xC0FFEE02, "c3": 0xC0FFEE03, "c4": 0xC0FFEE04,
         "kraus": 0xC0FFEE05}
CONFIG_N = {"c0": 12, "c1": 14, "c2": 16, "c3": 16, "c4": 17, "kraus": 16}


def _dp(a):
    return a.ctypes.data_as(nat.c_double_p)


def gaussian_entry(seed: int, counter: int) -> complex:
    out = np.zeros(2)
    nat.harness().hsg_gaussian_entry(seed, counter, _dp(out))
    return complex(out[0], out[1])


def uniform(seed: int, counter: int) -> float:
    return float(nat.harness().hsg_uniform(seed, counter))


def rank_psi(n: int, seed: int, rank: int = 4) -> np.ndarray:
    """psi_i[x] = gaussian_entry(seed + i, x), normalised; shape (rank, 2^n)."""
    psi = np.empty((rank, 1 << n), np.complex128)
    nat.harness().hsg_rank_psi(n, seed, rank, _dp(psi))
    return psi


def payload_count(n: int, m: int = 5) -> int:
    return int(nat.harness().hsg_payload_count(n, m))


def rho_payload(n: int, psi: np.ndarray, m: int = 5) -> np.ndarray:
    """Host tiled payload of rho = (1/rank) sum |psi_i><psi_i| (bit-identical to the device)."""
    psi = np.ascontiguousarray(psi, np.complex128)
    out = np.empty(payload_count(n, m), np.complex128)
    nat.harness().hsg_rho_payload(n, m, psi.shape[0], _dp(psi), _dp(out))
    return out


def rho_payload_range(n: int, psi: np.ndarray, t0: int, t1: int, m: int = 5) -> np.ndarray:
    psi = np.ascontiguousarray(psi, np.complex128)
    out = np.empty((t1 - t0) << (2 * m), np.complex128)
    nat.harness().hsg_rho_payload_range(n, m, psi.shape[0], _dp(psi), _dp(out), t0, t1)
    return out


def rho_payload_threaded(n: int, psi: np.ndarray, m: int = 5, out: np.ndarray | None = None,
                         threads: int | None = None) -> np.ndarray:
    """rho_payload over disjoint tile ranges on all host cores (ctypes releases the GIL)."""
    import os
    import threading
    psi = np.ascontiguousarray(psi, np.complex128)
    cnt = payload_count(n, m)
    if out is None:
        out = np.empty(cnt, np.complex128)
    G = (1 << n) >> m if n >= m else 1
    T = G * (G + 1) // 2
    threads = threads or os.cpu_count() or 1
    bounds = [T * i // threads for i in range(threads + 1)]
    L = nat.harness()

    def work(i):
        t0, t1 = bounds[i], bounds[i + 1]
        if t1 > t0:
            view = out[t0 << (2 * m): t1 << (2 * m)]
            L.hsg_rho_payload_range(n, m, psi.shape[0], _dp(psi), _dp(view), t0, t1)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return out


def haar(k: int, seed: int) -> np.ndarray:
    """Haar 2^k x 2^k unitary: QR (Gram-Schmidt) of a complex Gaussian, phase-fixed."""
    if not 0 <= k <= 6:
        raise ValueError("haar: k must be in [0, 6]")
    d = 1 << k
    u = np.empty((d, d), np.complex128)
    nat.harness().hsg_haar(k, seed, _dp(u))
    return u


def permutation(n: int, seed: int) -> list[int]:
    out = np.empty(n, np.uint32)
    nat.harness().hsg_permutation(n, seed, out.ctypes.data_as(nat.c_u32_p))
    return [int(v) for v in out]


def pauli_strings(n: int, count: int, seed: int):
    x = np.empty(count, np.uint64)
    z = np.empty(count, np.uint64)
    ny = np.empty(count, np.int32)
    coef = np.empty(count, np.float64)
    nat.harness().hsg_pauli_strings(n, count, seed, x.ctypes.data_as(nat.c_u64_p), z.ctypes.data_as(nat.c_u64_p),
                                    ny.ctypes.data_as(nat.c_i32_p), _dp(coef))
    return x, z, ny, coef


def pauli_payload(n: int, strings, m: int = 5) -> np.ndarray:
    x, z, ny, coef = strings
    out = np.empty(payload_count(n, m), np.complex128)
    nat.harness().hsg_pauli_payload(n, m, len(x), x.ctypes.data_as(nat.c_u64_p), z.ctypes.data_as(nat.c_u64_p),
                                    ny.ctypes.data_as(nat.c_i32_p), _dp(coef), _dp(out))
    return out


@dataclass
class Op:
    kind: str
    targets: tuple
    param: float = 0.0
    matrix: np.ndarray | None = field(default=None, repr=False)


def ops_c0(n: int = 12):
    """C0: Hadamard at every position 0..n-1 once."""
    return [Op("h", (q,)) for q in range(n)]


def ops_c1(n: int = 14, seed: int = SEEDS["c1"]):
    """C1: every ordered pair (i, j), i != j, i-major: CX(i -> j) then a fresh Haar U4 on (i, j)."""
    ops, idx = [], 0
    for i in range(n):
        for j in range(n):
            if i == j:
                continue
            ops.append(Op("cnot", (i, j)))
            ops.append(Op("unitary", (i, j), matrix=haar(2, seed + 1000 + idx)))
            idx += 1
    return ops


def ops_c2(n: int = 16):
    """C2: per qubit depolarising(p = 0.01) then amplitude damping(gamma = 0.05)."""
    ops = []
    for q in range(n):
        ops.append(Op("depol", (q,), 0.01))
        ops.append(Op("ampdamp", (q,), 0.05))
    return ops


def ops_c3(n: int = 16, layers: int = 20, seed: int = SEEDS["c3"]):
    """C3: per layer a seeded permutation cut into disjoint triples (one idle qubit when 3 does
    not divide n), each block O -> U^dagger O U with a Haar 8x8 U (dual channel {U^dagger})."""
    ops = []
    for layer in range(layers):
        perm = permutation(n, seed + 7919 * (layer + 1))
        for b in range(n // 3):
            tri = tuple(perm[3 * b: 3 * b + 3])
            ops.append(Op("unitary_dual", tri, matrix=haar(3, seed + 100000 + layer * 16 + b)))
    return ops


def matching_c4(n: int, seed: int, top: int = 3):
    """Seeded matching of n qubits into n // 2 pairs (one idle when n is odd) that matches every one
    of the top `top` qubits (idle never one of q14..q16)."""
    perm = permutation(n, seed)
    tops = set(range(n - top, n))
    idle = None
    if n % 2:
        idle = next(q for q in perm if q not in tops)
    rest = [q for q in perm if q != idle]
    return [(rest[2 * i], rest[2 * i + 1]) for i in range(len(rest) // 2)], idle


def ops_c4(n: int = 17, layers: int = 10, seed: int = SEEDS["c4"]):
    """C4: per layer Rz(theta_q) then H on each qubit, CX on a seeded matching including the top 3
    qubits, depolarising(0.001) on each qubit."""
    ops = []
    for layer in range(layers):
        for q in range(n):
            theta = 2.0 * math.pi * uniform(seed + layer, q)
            ops.append(Op("rz", (q,), theta))
            ops.append(Op("h", (q,)))
        pairs, _ = matching_c4(n, seed + 31 * (layer + 1))
        for a, b in pairs:
            ops.append(Op("cnot", (a, b)))
        for q in range(n):
            ops.append(Op("depol", (q,), 0.001))
    return ops


_PAULI = (np.eye(2, dtype=np.complex128), np.array([[0, 1], [1, 0]], np.complex128),
          np.array([[0, -1j], [1j, 0]], np.complex128), np.array([[1, 0], [0, -1]], np.complex128))


def depolarising2_ops(p: float) -> np.ndarray:
    """Two-qubit depolarising channel: sqrt(1 - p) I4 and sqrt(p / 15) P_a (x) P_b for the 15
    non-identity Pauli pairs (rank 16; built with make_generic, not a reference library entry)."""
    ops = []
    for a in range(4):
        for b in range(4):
            w = math.sqrt(1.0 - p) if a == b == 0 else math.sqrt(p / 15.0)
            ops.append(w * np.kron(_PAULI[a], _PAULI[b]))
    return np.stack(ops)


def random_kraus_ops(k: int, rank: int, seed: int) -> np.ndarray:
    """Seeded trace-preserving Kraus set of `rank` operators on k qubits: a random isometry V of
    (rank * 2^k) x 2^k (V^dagger V = I, Gram-Schmidt of a complex Gaussian) cut into rank blocks of
    2^k rows, so sum_a K_a^dagger K_a = I."""
    d = 1 << k
    v = np.empty((rank * d, d), np.complex128)
    if nat.harness().hsg_isometry(rank * d, d, seed, _dp(v)) != 0:
        raise ValueError("random_kraus_ops: invalid shape")
    return v.reshape(rank, d, d)


def ops_kraus(n: int = 16, layers: int = 2, seed: int = SEEDS["kraus"]):
    """Generic Kraus channels of rank > 1 (the north_star's Kraus-channel sum beyond the library's
    single-qubit channels; VERDICT r1 'next' #2).  Per layer: a seeded permutation of the qubits cut
    into pairs, each pair a two-qubit depolarising channel (p = 0.01, rank 16); a second permutation
    cut into disjoint triples, each a seeded random rank-4 three-qubit channel.  n = 16: 2 x (8 + 5)
    = 26 channel passes."""
    ops = []
    for layer in range(layers):
        perm = permutation(n, seed + 7919 * (layer + 1))
        for b in range(n // 2):
            ops.append(Op("kraus", (perm[2 * b], perm[2 * b + 1]), 0.01, matrix=depolarising2_ops(0.01)))
        perm = permutation(n, seed + 104729 * (layer + 1))
        for b in range(n // 3):
            ops.append(Op("kraus", tuple(perm[3 * b: 3 * b + 3]),
                          matrix=random_kraus_ops(3, 4, seed + 1000 * (layer + 1) + b)))
    return ops


def config_ops(name: str, n: int | None = None):
    n = n if n is not None else CONFIG_N[name]
    return {"c0": ops_c0, "c1": ops_c1, "c2": ops_c2, "c3": ops_c3, "c4": ops_c4, "kraus": ops_kraus}[name](n)


def amplitude_damping_ops(gamma: float) -> np.ndarray:
    return np.stack([np.array([[1, 0], [0, math.sqrt(1 - gamma)]], np.complex128),
                     np.array([[0, math.sqrt(gamma)], [0, 0]], np.complex128)])
