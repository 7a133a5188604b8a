"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loaded only by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg, always as the *checker* (or the reference arm being timed),
never as the thing measured for the product.  The product package
``paper_2604_15765_b200`` never imports this module.

Two CPU engines are exposed:

* ``Oracle`` -- our C restatement of the reference path (``oracle/orkan_oracle.c``,
  built into ``oracle/_ref/liborkan_oracle.so``).
* ``Reference`` -- the reference library itself (arXiv 2604.15765, ``/root/reference/proj``),
  compiled from its own sources by ``oracle/build_ref.sh`` into ``oracle/_ref/libhermsim_ref.so``
  (with the documented kernels.cpp:365/367/369 fix; ``patched=False`` loads the unpatched build).

The gate library below restates ``channel.cpp:82-154`` (depolarising, native_gate) as plain
data so both engines are driven with identical channel descriptions.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

# GateKind (channel.hpp:36) and KernelPath (kernels.hpp:12-24)
GENERIC, PAULI_X, PAULI_Y, PHASE, HADAMARD, PERM = range(6)
KERNEL_PATHS = [
    "dense-generic", "packed-generic", "tiled-intra", "tiled-cross", "tiled-mixed", "dense-fallback",
    "native-pauli-x", "native-pauli-y", "native-phase", "native-hadamard", "native-permutation",
]

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_dp = ctypes.POINTER(ctypes.c_double)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _u32(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a, a.ctypes.data_as(_u32p)


@dataclass
class Channel:
    """ChannelSpec restated as data (channel.hpp:41-50)."""

    name: str
    kind: int
    ops: np.ndarray  # (nops, d, d) complex128, constructor order
    phases: np.ndarray = field(default_factory=lambda: np.ones(2, np.complex128))
    perm: np.ndarray | None = None  # (d,) uint32, constructor order
    theta: float = 0.0  # rz angle (native_gate argument)

    @property
    def k(self) -> int:
        return int(round(math.log2(self.ops.shape[1])))


def _m2(a, b, c, d):
    return np.array([[a, b], [c, d]], np.complex128)


def _perm_mat(k, table):
    d = 1 << k
    m = np.zeros((d, d), np.complex128)
    for col in range(d):
        m[table[col], col] = 1.0
    return m


def native_gate(name: str, theta: float = 0.0) -> Channel:
    """native_gate (channel.cpp:95-154)."""
    if name == "x":
        return Channel("x", PAULI_X, _m2(0, 1, 1, 0)[None])
    if name == "y":
        return Channel("y", PAULI_Y, _m2(0, -1j, 1j, 0)[None])
    if name == "z":
        return Channel("z", PHASE, _m2(1, 0, 0, -1)[None], np.array([1, -1], np.complex128))
    if name == "s":
        return Channel("s", PHASE, _m2(1, 0, 0, 1j)[None], np.array([1, 1j], np.complex128))
    if name == "t":
        p1 = complex(math.cos(math.pi / 4), math.sin(math.pi / 4))
        return Channel("t", PHASE, _m2(1, 0, 0, p1)[None], np.array([1, p1], np.complex128))
    if name == "rz":
        p0 = complex(math.cos(-theta / 2), math.sin(-theta / 2))
        p1 = complex(math.cos(theta / 2), math.sin(theta / 2))
        return Channel("rz", PHASE, _m2(p0, 0, 0, p1)[None], np.array([p0, p1], np.complex128), theta=theta)
    if name == "h":
        r = 1.0 / math.sqrt(2.0)
        return Channel("h", HADAMARD, _m2(r, r, r, -r)[None])
    tables = {"cnot": (2, [0, 1, 3, 2]), "swap": (2, [0, 2, 1, 3]), "toffoli": (3, [0, 1, 2, 3, 4, 5, 7, 6])}
    if name in tables:
        k, t = tables[name]
        return Channel(name, PERM, _perm_mat(k, t)[None], perm=np.array(t, np.uint32))
    raise ValueError(f"unknown gate name: {name}")


def depolarising(p: float) -> Channel:
    """depolarising (channel.cpp:82-93): sqrt(1-p) I, sqrt(p/3) X, Y, Z."""
    w0, w = math.sqrt(1.0 - p), math.sqrt(p / 3.0)
    ops = np.stack([w0 * _m2(1, 0, 0, 1), w * _m2(0, 1, 1, 0), w * _m2(0, -1j, 1j, 0), w * _m2(1, 0, 0, -1)])
    return Channel("depolarising", GENERIC, ops)


def amplitude_damping(gamma: float) -> Channel:
    """Not in the reference library: make_generic of K0, K1."""
    ops = np.stack([_m2(1, 0, 0, math.sqrt(1.0 - gamma)), _m2(0, math.sqrt(gamma), 0, 0)])
    return Channel("amplitude_damping", GENERIC, ops)


def generic(ops, name="generic") -> Channel:
    ops = np.ascontiguousarray(np.asarray(ops, np.complex128))
    if ops.ndim == 2:
        ops = ops[None]
    return Channel(name, GENERIC, ops)


def dual(ch: Channel) -> Channel:
    """dual_channel (channel.cpp:188-194): {L^dagger}; kind becomes generic."""
    return Channel(ch.name + "^dual", GENERIC, np.ascontiguousarray(np.conj(np.transpose(ch.ops, (0, 2, 1)))))


def payload_count(n: int, m: int) -> int:
    dim, edge = 1 << n, 1 << m
    grid = dim // edge if dim >= edge else 1
    return grid * (grid + 1) // 2 * edge * edge


class Oracle:
    """ctypes binding of oracle/orkan_oracle.c."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(REF_DIR, "liborkan_oracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        L = self.lib = ctypes.CDLL(path)
        L.or_apply.restype = ctypes.c_int
        L.or_apply.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp,
                               _u32p, _u32p, ctypes.c_int, _u64p]
        L.or_expectation.restype = ctypes.c_double
        L.or_expectation.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int]
        L.or_frobenius.restype = ctypes.c_double
        L.or_frobenius.argtypes = [_dp, ctypes.c_int, ctypes.c_int]
        L.or_gaussian_entry.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _dp]
        L.or_insert_bits.restype = ctypes.c_uint64
        L.or_insert_bits.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u32p, ctypes.c_int]
        L.or_tile_offset.restype = ctypes.c_uint64
        L.or_tile_offset.argtypes = [ctypes.c_uint64] * 3
        L.or_payload_count.restype = ctypes.c_uint64
        L.or_payload_count.argtypes = [ctypes.c_int, ctypes.c_int]
        L.or_tiled_to_dense.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp]
        L.or_dense_to_tiled.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp]
        L.or_dense_kraus_apply.restype = ctypes.c_int
        L.or_dense_kraus_apply.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _u32p]
        L.or_transfer_from_kraus.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp]

    def apply(self, payload: np.ndarray, n: int, m: int, ch: Channel, targets, allow_native=True):
        assert payload.dtype == np.complex128 and payload.flags.c_contiguous
        ops = np.ascontiguousarray(ch.ops, np.complex128)
        ph = np.ascontiguousarray(ch.phases, np.complex128)
        tg, tgp = _u32(targets)
        perm = None
        if ch.perm is not None:
            perm, permp = _u32(ch.perm)
        else:
            permp = None
        sub = np.zeros(3, np.uint64)
        path = self.lib.or_apply(_dptr(payload), n, m, ch.kind, ch.k, ops.shape[0], _dptr(ops), _dptr(ph), permp,
                                 tgp, 1 if allow_native else 0, sub.ctypes.data_as(_u64p))
        if path < 0:
            raise ValueError(f"oracle apply failed ({path})")
        return KERNEL_PATHS[path], tuple(int(x) for x in sub)

    def expectation(self, rho, obs, n, m) -> float:
        return self.lib.or_expectation(_dptr(rho), _dptr(obs), n, m)

    def frobenius(self, payload, n, m) -> float:
        return self.lib.or_frobenius(_dptr(payload), n, m)

    def gaussian_entry(self, seed, counter) -> complex:
        out = np.zeros(2)
        self.lib.or_gaussian_entry(seed, counter, _dptr(out))
        return complex(out[0], out[1])

    def insert_bits(self, s, a, pos) -> int:
        p, pp = _u32(pos)
        return int(self.lib.or_insert_bits(s, a, pp, len(p)))

    def tile_offset(self, ti, tj, M) -> int:
        return int(self.lib.or_tile_offset(ti, tj, M))

    def to_dense(self, payload, n, m) -> np.ndarray:
        d = np.zeros((1 << n, 1 << n), np.complex128)
        self.lib.or_tiled_to_dense(_dptr(payload), n, m, _dptr(d))
        return d

    def from_dense(self, dense, n, m) -> np.ndarray:
        p = np.zeros(payload_count(n, m), np.complex128)
        d = np.ascontiguousarray(dense, np.complex128)
        self.lib.or_dense_to_tiled(_dptr(d), n, m, _dptr(p))
        return p

    def dense_kraus_apply(self, dense, n, ch: Channel, targets) -> np.ndarray:
        d = np.ascontiguousarray(dense, np.complex128).copy()
        ops = np.ascontiguousarray(ch.ops, np.complex128)
        tg, tgp = _u32(targets)
        rc = self.lib.or_dense_kraus_apply(_dptr(d), n, ch.k, ops.shape[0], _dptr(ops), tgp)
        if rc != 0:
            raise MemoryError("dense oracle allocation failed")
        return d

    def transfer_from_kraus(self, ops) -> np.ndarray:
        ops = np.ascontiguousarray(ops, np.complex128)
        k = int(round(math.log2(ops.shape[1])))
        s = np.zeros((4 ** k, 4 ** k), np.complex128)
        self.lib.or_transfer_from_kraus(k, ops.shape[0], _dptr(ops), _dptr(s))
        return s


class Reference:
    """ctypes binding of the compiled reference (oracle/ref_capi.cpp over hermsim::apply)."""

    def __init__(self, patched: bool = True, path: str | None = None):
        name = "libhermsim_ref.so" if patched else "libhermsim_ref_unpatched.so"
        path = path or os.path.join(REF_DIR, name)
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference library missing: {path} (run `make -C oracle ref` where "
                                    "/root/reference is mounted)")
        L = self.lib = ctypes.CDLL(path)
        L.ref_tiled_create.restype = ctypes.c_void_p
        L.ref_tiled_create.argtypes = [ctypes.c_int, ctypes.c_int]
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_payload.restype = _dp
        L.ref_payload.argtypes = [ctypes.c_void_p]
        L.ref_payload_count.restype = ctypes.c_uint64
        L.ref_payload_count.argtypes = [ctypes.c_void_p]
        L.ref_last_error.restype = ctypes.c_char_p
        sub = [_u64p]
        L.ref_apply_native.restype = ctypes.c_int
        L.ref_apply_native.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_double, _u32p, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int] + sub
        L.ref_apply_depolarising.restype = ctypes.c_int
        L.ref_apply_depolarising.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_uint32, ctypes.c_int] + sub
        L.ref_apply_generic.restype = ctypes.c_int
        L.ref_apply_generic.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _dp, _u32p, ctypes.c_int,
                                        ctypes.c_int] + sub
        L.ref_gaussian_entry.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _dp]
        L.ref_footprint_bytes.restype = ctypes.c_uint64
        L.ref_footprint_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.ref_insert_bits.restype = ctypes.c_uint64
        L.ref_insert_bits.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u32p, ctypes.c_int]
        L.ref_tile_offset.restype = ctypes.c_uint64
        L.ref_tile_offset.argtypes = [ctypes.c_uint64] * 3
        L.ref_random_hermitian.restype = ctypes.c_void_p
        L.ref_random_hermitian.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
        L.ref_save.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.ref_convert.restype = ctypes.c_void_p
        L.ref_convert.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.ref_dense_create.restype = ctypes.c_void_p
        L.ref_dense_create.argtypes = [ctypes.c_int]
        L.ref_format.restype = ctypes.c_int
        L.ref_format.argtypes = [ctypes.c_void_p]
        L.ref_load.restype = ctypes.c_void_p
        L.ref_load.argtypes = [ctypes.c_char_p]

    # -- state handles -------------------------------------------------------------------
    def create(self, n: int, m: int = 5, payload: np.ndarray | None = None):
        h = self.lib.ref_tiled_create(n, m)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        if payload is not None:
            self.view(h)[:] = payload
        return h

    def view(self, h) -> np.ndarray:
        cnt = int(self.lib.ref_payload_count(h))
        ptr = self.lib.ref_payload(h)
        return np.ctypeslib.as_array(ptr, shape=(2 * cnt,)).view(np.complex128)

    def free(self, h):
        self.lib.ref_free(h)

    def save(self, h, path: str):
        if self.lib.ref_save(h, path.encode()):
            raise IOError(self.lib.ref_last_error().decode())

    def load(self, path: str):
        h = self.lib.ref_load(path.encode())
        if not h:
            raise IOError(self.lib.ref_last_error().decode())
        return h

    def create_dense(self, n: int, dense: np.ndarray | None = None):
        h = self.lib.ref_dense_create(n)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        if dense is not None:
            self.view(h)[:] = np.ascontiguousarray(dense, np.complex128).reshape(-1)
        return h

    def convert(self, h, fmt: str, m: int = 5):
        """hermsim::convert(h, format, m) into a new handle (free it with free())."""
        out = self.lib.ref_convert(h, {"dense": 0, "packed": 1, "tiled": 2}[fmt], m)
        if not out:
            raise ValueError(self.lib.ref_last_error().decode())
        return out

    def random_hermitian(self, n, seed, m=5):
        h = self.lib.ref_random_hermitian(n, seed, 2, m)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return h

    # -- hermsim::apply ------------------------------------------------------------------
    def apply(self, h, ch: Channel, targets, threads: int = 1, allow_native: bool = True):
        tg, tgp = _u32(targets)
        sub = np.zeros(3, np.uint64)
        subp = sub.ctypes.data_as(_u64p)
        if ch.kind != GENERIC:
            path = self.lib.ref_apply_native(h, ch.name.encode(), ch.theta, tgp, len(tg), threads,
                                             1 if allow_native else 0, subp)
        elif ch.name == "depolarising":
            path = self.lib.ref_apply_generic(h, 1, 4, _dptr(np.ascontiguousarray(ch.ops)), tgp, threads, 0, subp)
        else:
            ops = np.ascontiguousarray(ch.ops, np.complex128)
            path = self.lib.ref_apply_generic(h, ch.k, ops.shape[0], _dptr(ops), tgp, threads, 0, subp)
        if path < 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return KERNEL_PATHS[path], tuple(int(x) for x in sub)

    def gaussian_entry(self, seed, counter) -> complex:
        out = np.zeros(2)
        self.lib.ref_gaussian_entry(seed, counter, _dptr(out))
        return complex(out[0], out[1])

    def footprint_bytes(self, n, m, fmt=2) -> int:
        return int(self.lib.ref_footprint_bytes(n, m, fmt))

    def insert_bits(self, s, a, pos) -> int:
        p, pp = _u32(pos)
        return int(self.lib.ref_insert_bits(s, a, pp, len(p)))

    def tile_offset(self, ti, tj, M) -> int:
        return int(self.lib.ref_tile_offset(ti, tj, M))


def rel_max_err(got: np.ndarray, want: np.ndarray, fro: float) -> float:
    """max elementwise |delta| / ||want||_F (SURVEY 8c tolerance metric)."""
    return float(np.max(np.abs(got - want)) / max(fro, 1e-300))
