"""Python mirror of the reference's public API (arXiv 2604.15765, ``/root/reference/proj/include/
hermsim``), backed by the B200 engine.

Same names, argument meaning and error behaviour as the C++ reference, so the parity tests read
like the reference's own (SPEC.md acceptance criteria):

======================================  ===================================================
reference (hermsim::)                   here
======================================  ===================================================
TiledHermitian(n, m)  storage.hpp:60    TiledHermitian(n, m, device) -- payload in HBM
native_gate / depolarising /            native_gate / depolarising / make_generic /
make_generic / dual_channel             dual_channel  (C++ host layer via hermsim_b200_c.h)
bind_channel  channel.cpp:196-268       bind_channel
validate_cptni channel.cpp:168-186      validate_cptni
apply(h, spec, targets, opts)           apply(h, spec, targets, opts) -> ApplyPlan
  kernels.cpp:510-549
(absent) tr(rho O)                      expectation(rho, obs)
======================================  ===================================================

Exceptions: ``ValueError`` where the reference throws ``std::invalid_argument``, ``IndexError``
for ``std::out_of_range``.  There is no CPU path: every operation runs the CUDA engine.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat

KERNEL_PATHS = [
    "dense-generic", "packed-generic", "tiled-intra", "tiled-cross", "tiled-mixed", "dense-fallback",
    "native-pauli-x", "native-pauli-y", "native-phase", "native-hadamard", "native-permutation",
]
GATE_KINDS = ["generic_kraus", "pauli_x", "pauli_y", "diagonal_phase", "hadamard", "permutation"]


def _dp(a: np.ndarray):
    return a.ctypes.data_as(nat.c_double_p)


def _u32(seq):
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.uint32))
    return a, a.ctypes.data_as(nat.c_u32_p)


def footprint_bytes(n: int, tile_exp: int = 5) -> int:
    """footprint_bytes(n, m, tiled) (storage.cpp:294-310)."""
    if n < 1 or n > 30:
        raise ValueError("qubit count must be in [1, 30]")
    if tile_exp < 0 or tile_exp > n + 2:
        raise ValueError("tile exponent must be in [0, n + 2]")
    dim, edge = 1 << n, 1 << tile_exp
    grid = dim // edge if dim >= edge else 1
    return grid * (grid + 1) // 2 * edge * edge * 16


class TiledHermitian:
    """Lower-triangle tile storage in HBM (storage.hpp:60-96); payload layout identical."""

    default_tile_exp = 5

    def __init__(self, n_qubits: int, tile_exp: int = 5, device: int = 0, nshards: int = 1, shard: int = 0):
        """nshards > 1: this object holds shard `shard` of the operator (multigpu.py)."""
        L = nat.engine()
        h = ctypes.c_void_p()
        nat.check(L.hs_state_create_sharded(n_qubits, tile_exp, device, nshards, shard, ctypes.byref(h)),
                  "TiledHermitian")
        self.nshards, self.shard = nshards, shard
        self._h = h
        self._n, self._m = n_qubits, tile_exp
        cnt, grid = ctypes.c_uint64(), ctypes.c_uint64()
        nat.check(L.hs_state_info(h, None, None, ctypes.byref(cnt), ctypes.byref(grid)))
        self._count, self._grid = int(cnt.value), int(grid.value)
        self.device = device

    # -- shape (storage.hpp:70-84)
    def qubits(self) -> int:
        return self._n

    def tile_exp(self) -> int:
        return self._m

    def dim(self) -> int:
        return 1 << self._n

    def tile_edge(self) -> int:
        return 1 << self._m

    def grid_dim(self) -> int:
        return self._grid

    def tile_count(self) -> int:
        return self._grid * (self._grid + 1) // 2

    def element_count(self) -> int:
        return self._count

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("state has been freed")
        return self._h

    # -- host <-> HBM
    def upload(self, payload: np.ndarray) -> None:
        p = np.ascontiguousarray(payload, dtype=np.complex128)
        if p.size != self._count:
            raise ValueError("payload length mismatch")
        nat.check(nat.engine().hs_state_upload(self.handle, _dp(p), self._count), "upload")

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self._count, np.complex128)
        nat.check(nat.engine().hs_state_download(self.handle, _dp(out), self._count), "download")
        return out

    def download_range(self, offset: int, count: int, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(count, np.complex128)
        elif out.dtype != np.complex128 or out.size != count or not out.flags.c_contiguous:
            raise ValueError("download_range: out must be a contiguous complex128 array of `count` elements")
        nat.check(nat.engine().hs_state_download_range(self.handle, _dp(out), offset, count), "download")
        return out

    def upload_range(self, payload: np.ndarray, offset: int) -> None:
        p = np.ascontiguousarray(payload, dtype=np.complex128)
        nat.check(nat.engine().hs_state_upload_range(self.handle, _dp(p), offset, p.size), "upload")

    def copy_from(self, other: "TiledHermitian") -> None:
        nat.check(nat.engine().hs_state_copy(self.handle, other.handle), "copy")

    def zero(self) -> None:
        nat.check(nat.engine().hs_state_zero(self.handle), "zero")

    def synchronize(self) -> None:
        nat.check(nat.engine().hs_state_synchronize(self.handle), "synchronize")

    def fill_mixture(self, psi: np.ndarray) -> None:
        """rho = (1/rank) sum_i |psi_i><psi_i| built on the device (bit-identical to the host)."""
        psi = np.ascontiguousarray(psi, np.complex128)
        nat.check(nat.engine().hs_state_fill_mixture(self.handle, psi.shape[0], _dp(psi)), "fill_mixture")

    def fill_pauli_sum(self, x, z, ny, coef) -> None:
        x = np.ascontiguousarray(x, np.uint64)
        z = np.ascontiguousarray(z, np.uint64)
        ny = np.ascontiguousarray(ny, np.int32)
        coef = np.ascontiguousarray(coef, np.float64)
        nat.check(nat.engine().hs_state_fill_pauli_sum(
            self.handle, len(x), x.ctypes.data_as(nat.c_u64_p), z.ctypes.data_as(nat.c_u64_p),
            ny.ctypes.data_as(nat.c_i32_p), _dp(coef)), "fill_pauli_sum")

    def distance_to_mixture(self, psi: np.ndarray) -> float:
        """max |stored element - (1/rank) sum |psi_i><psi_i|| over the payload (device-side)."""
        psi = np.ascontiguousarray(psi, np.complex128)
        out = ctypes.c_double()
        nat.check(nat.engine().hs_state_distance_mixture(self.handle, psi.shape[0], _dp(psi), ctypes.byref(out)),
                  "distance_to_mixture")
        return out.value

    def fill_random_hermitian(self, seed: int) -> None:
        """hermsim::random_hermitian(n, seed, tiled, m) (storage.cpp:195-201), generated on the device."""
        nat.check(nat.engine().hs_state_fill_random_hermitian(self.handle, seed), "random_hermitian")

    def fill_basis_projector(self, basis: int) -> None:
        """hermsim::basis_projector(n, basis, tiled, m) (storage.cpp:230-239)."""
        nat.check(nat.engine().hs_state_fill_basis_projector(self.handle, basis), "basis_projector")

    # -- format conversions on the device (hermsim::to_dense / convert, storage.cpp:241-292) ------
    def to_dense(self, out: np.ndarray | None = None) -> np.ndarray:
        """hermsim::to_dense: the N x N row-major matrix (bit-identical to the reference's)."""
        N = self.dim()
        if out is None:
            out = np.empty((N, N), np.complex128)
        if out.shape != (N, N) or out.dtype != np.complex128 or not out.flags.c_contiguous:
            raise ValueError("to_dense: out must be a C-contiguous (N, N) complex128 array")
        nat.check(nat.engine().hs_state_to_dense(self.handle, out.ctypes.data, 0), "to_dense")
        return out

    def to_packed(self, out: np.ndarray | None = None) -> np.ndarray:
        """convert(h, packed): the column-major packed lower triangle, N(N+1)/2 elements."""
        N = self.dim()
        cnt = N * (N + 1) // 2
        if out is None:
            out = np.empty(cnt, np.complex128)
        if out.shape != (cnt,) or out.dtype != np.complex128 or not out.flags.c_contiguous:
            raise ValueError("to_packed: out must be a contiguous complex128 array of N(N+1)/2 elements")
        nat.check(nat.engine().hs_state_to_packed(self.handle, out.ctypes.data, 0), "to_packed")
        return out

    def from_dense(self, dense: np.ndarray) -> None:
        """convert(MatrixHandle(dense), tiled, m): stored (i >= j) = d(i, j), diagonal-tile upper halves
        = conj(d(j, i))."""
        N = self.dim()
        d = np.ascontiguousarray(dense, np.complex128)
        if d.shape != (N, N):
            raise ValueError("from_dense: shape must be (N, N)")
        nat.check(nat.engine().hs_state_from_dense(self.handle, d.ctypes.data, 0), "from_dense")

    def from_packed(self, packed: np.ndarray) -> None:
        """convert(MatrixHandle(packed), tiled, m)."""
        N = self.dim()
        p = np.ascontiguousarray(packed, np.complex128)
        if p.shape != (N * (N + 1) // 2,):
            raise ValueError("from_packed: need N(N+1)/2 elements")
        nat.check(nat.engine().hs_state_from_packed(self.handle, p.ctypes.data, 0), "from_packed")

    def save(self, path: str) -> None:
        """hermsim::save (storage_io.cpp:34-56): OHRM container, tiled format."""
        nat.check(nat.engine().hs_state_save(self.handle, os.fsencode(path)), "save")

    @classmethod
    def load(cls, path: str, device: int = 0) -> "TiledHermitian":
        """hermsim::load (storage_io.cpp:58-118) of a tiled OHRM file into HBM."""
        h = ctypes.c_void_p()
        nat.check(nat.engine().hs_state_load(os.fsencode(path), device, ctypes.byref(h)), "load")
        self = cls.__new__(cls)
        L = nat.engine()
        n, m = ctypes.c_int(), ctypes.c_int()
        cnt, grid = ctypes.c_uint64(), ctypes.c_uint64()
        nat.check(L.hs_state_info(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(cnt), ctypes.byref(grid)))
        self.nshards, self.shard, self._h = 1, 0, h
        self._n, self._m = n.value, m.value
        self._count, self._grid = int(cnt.value), int(grid.value)
        self.device = device
        return self

    def free(self) -> None:
        if getattr(self, "_h", None) is not None:
            nat.engine().hs_state_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()


class ChannelSpec:
    """ChannelSpec (channel.hpp:41-50) owned by the C++ host layer."""

    def __init__(self, handle, name: str = ""):
        self._c = handle
        L = nat.engine()
        kind, k, nops = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        nat.check(L.hb_channel_info(handle, ctypes.byref(kind), ctypes.byref(k), ctypes.byref(nops)), facade=True)
        self.kind = GATE_KINDS[kind.value]
        self.k, self.nops, self.name = k.value, nops.value, name

    def locality(self) -> int:
        return self.k

    @property
    def kraus(self) -> np.ndarray:
        d = 1 << self.k
        out = np.empty((self.nops, d, d), np.complex128)
        nat.check(nat.engine().hb_channel_kraus(self._c, _dp(out)), facade=True)
        return out

    @property
    def transfer(self) -> np.ndarray:
        d2 = 1 << (2 * self.k)
        out = np.empty((d2, d2), np.complex128)
        nat.check(nat.engine().hb_channel_transfer(self._c, _dp(out)), facade=True)
        return out

    @property
    def phases(self) -> np.ndarray:
        out = np.empty(2, np.complex128)
        nat.check(nat.engine().hb_channel_phases(self._c, _dp(out)), facade=True)
        return out

    @property
    def perm(self) -> np.ndarray | None:
        L = nat.engine()
        cnt = L.hb_channel_perm(self._c, None)
        if cnt <= 0:
            return None
        out = np.empty(cnt, np.uint32)
        L.hb_channel_perm(self._c, out.ctypes.data_as(nat.c_u32_p))
        return out

    def __del__(self):
        try:
            if getattr(self, "_c", None) is not None:
                nat.engine().hb_channel_free(self._c)
                self._c = None
        except Exception:
            pass


def _new_channel(fn, *args, name="") -> ChannelSpec:
    h = ctypes.c_void_p()
    nat.check(fn(*args, ctypes.byref(h)), name, facade=True)
    return ChannelSpec(h, name)


def native_gate(name: str, theta: float = 0.0) -> ChannelSpec:
    """native_gate (channel.cpp:95-154): x y z s t rz h cnot swap toffoli."""
    return _new_channel(nat.engine().hb_channel_native, name.encode(), float(theta), name=name)


def depolarising(p: float) -> ChannelSpec:
    """depolarising (channel.cpp:82-93)."""
    return _new_channel(nat.engine().hb_channel_depolarising, float(p), name="depolarising")


def make_generic(name: str, ops, validate: bool = False, tol: float = 1e-10) -> ChannelSpec:
    """make_generic(name, make_kraus_set(k, ops)) (channel.cpp:10-22,73-80)."""
    ops = np.ascontiguousarray(np.asarray(ops, np.complex128))
    if ops.ndim == 2:
        ops = ops[None]
    if ops.ndim != 3 or ops.shape[1] != ops.shape[2]:
        raise ValueError("Kraus set: operator dimension mismatch")
    d = ops.shape[1]
    k = d.bit_length() - 1
    if (1 << k) != d:
        raise ValueError("Kraus set: operator dimension mismatch")
    return _new_channel(nat.engine().hb_channel_generic, name.encode(), k, ops.shape[0], _dp(ops),
                        1 if validate else 0, float(tol), name=name)


def amplitude_damping(gamma: float) -> ChannelSpec:
    """Not in the reference library: make_generic of K0, K1."""
    k0 = np.array([[1, 0], [0, np.sqrt(1 - gamma)]], np.complex128)
    k1 = np.array([[0, np.sqrt(gamma)], [0, 0]], np.complex128)
    return make_generic("amplitude_damping", np.stack([k0, k1]))


def dual_channel(spec: ChannelSpec) -> ChannelSpec:
    """make_generic(dual_channel(kraus)) -- Heisenberg picture (channel.cpp:188-194)."""
    return _new_channel(nat.engine().hb_channel_dual, spec._c, name=spec.name + "^dual")


def bind_channel(spec: ChannelSpec, targets):
    """bind_channel (channel.cpp:196-268) -> (sorted qubits, bound Kraus ops, bound perm)."""
    tg, tgp = _u32(targets)
    d = 1 << spec.k
    sorted_q = np.zeros(3, np.uint32)
    ops = np.empty((spec.nops, d, d), np.complex128)
    perm = np.zeros(8, np.uint32)
    nat.check(nat.engine().hb_bind(spec._c, tgp, len(tg), sorted_q.ctypes.data_as(nat.c_u32_p), _dp(ops),
                                   perm.ctypes.data_as(nat.c_u32_p)), "bind_channel", facade=True)
    has_perm = spec.perm is not None
    return sorted_q[:len(tg)].copy(), ops, (perm[:d].copy() if has_perm else None)


def validate_cptni(spec: ChannelSpec, tol: float = 1e-10):
    """validate_cptni (channel.cpp:168-186) -> (classification, max_deviation, min_eigenvalue)."""
    c, md, me = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    nat.check(nat.engine().hb_validate_cptni(spec._c, tol, ctypes.byref(c), ctypes.byref(md), ctypes.byref(me)),
              facade=True)
    return ["trace_preserving", "trace_non_increasing", "invalid"][c.value], md.value, me.value


@dataclass
class ApplyOptions:
    """ApplyOptions (kernels.hpp:43-46); ``threads`` is accepted and ignored (CUDA grid)."""

    threads: int = 1
    allow_native: bool = True
    count_subcases: bool = True


@dataclass
class ApplyPlan:
    """ApplyPlan (kernels.hpp:48-52)."""

    path: str
    targets: tuple
    subcases: tuple = field(default=(0, 0, 0))
    touched_bytes: int = 0  # HBM bytes read + written by the launch (extension of the reference plan)


def apply(h: TiledHermitian, spec: ChannelSpec, targets, opts: ApplyOptions | None = None) -> ApplyPlan:
    """hermsim::apply (kernels.hpp:58-61): targets in constructor order (controls first)."""
    opts = opts or ApplyOptions()
    tg, tgp = _u32(targets)
    plan = nat.HsPlan()
    nat.check(nat.engine().hb_apply(h.handle, spec._c, tgp, len(tg), 1 if opts.allow_native else 0,
                                    1 if opts.count_subcases else 0, ctypes.byref(plan)), "apply", facade=True)
    return ApplyPlan(KERNEL_PATHS[plan.path], tuple(plan.targets[: plan.k]), tuple(plan.subcases),
                     int(plan.touched_bytes))


class Graph:
    """A captured sequence of operations on one state (CUDA graph); `launch()` replays it on the
    state's stream.  Build with `capture(state)`:

        with hermsim.capture(rho) as g:
            for spec, tg in circuit:
                hermsim.apply(rho, spec, tg)
        g.launch(); g.launch()
    """

    def __init__(self, state: TiledHermitian):
        self.state = state
        self._g = None

    def __enter__(self):
        nat.check(nat.engine().hs_graph_begin(self.state.handle), "graph begin")
        return self

    def __exit__(self, exc_type, exc, tb):
        g = ctypes.c_void_p()
        rc = nat.engine().hs_graph_end(self.state.handle, ctypes.byref(g))
        if exc_type is None:
            nat.check(rc, "graph end")
            self._g = g
        return False

    def nodes(self) -> int:
        out = ctypes.c_uint64()
        nat.check(nat.engine().hs_graph_nodes(self._g, ctypes.byref(out)), "graph nodes")
        return int(out.value)

    def launch(self) -> None:
        nat.check(nat.engine().hs_graph_launch(self._g, self.state.handle), "graph launch")

    def __del__(self):
        try:
            if self._g is not None:
                nat.engine().hs_graph_free(self._g)
                self._g = None
        except Exception:
            pass


def capture(state: TiledHermitian) -> Graph:
    return Graph(state)


def convert(h: TiledHermitian, target: str = "tiled", tile_exp: int = 5):
    """hermsim::convert (storage.cpp:285-292) on the device.  target "tiled" returns a new
    TiledHermitian with tile exponent `tile_exp` on the same device; "dense" / "packed" return the
    host array of that format (the reference's DenseHermitian / PackedHermitian payloads)."""
    if target == "dense":
        return h.to_dense()
    if target == "packed":
        return h.to_packed()
    if target != "tiled":
        raise ValueError(f"convert: unknown format '{target}'")
    out = TiledHermitian(h.qubits(), tile_exp, device=h.device)
    h.synchronize()
    nat.check(nat.engine().hs_state_convert(h.handle, out.handle), "convert")
    return out


def to_dense(h: TiledHermitian) -> np.ndarray:
    """hermsim::to_dense (storage.cpp:241-283)."""
    return h.to_dense()


def expectation(rho: TiledHermitian, obs: TiledHermitian) -> float:
    """tr(rho O) (strict ti > tj per SPEC.md); deterministic reduction."""
    out = ctypes.c_double()
    nat.check(nat.engine().hs_expectation(rho.handle, obs.handle, ctypes.byref(out)), "expectation")
    return out.value


def trace(h: TiledHermitian) -> float:
    out = ctypes.c_double()
    nat.check(nat.engine().hs_trace(h.handle, ctypes.byref(out)), "trace")
    return out.value


def frobenius(h: TiledHermitian) -> float:
    """Logical Frobenius norm sqrt(sum_diag |x|^2 + 2 sum_offdiag |x|^2)."""
    out = ctypes.c_double()
    nat.check(nat.engine().hs_frobenius(h.handle, ctypes.byref(out)), "frobenius")
    return out.value


# ---- bound engine entry points (targets ascending, local bit l <-> targets[l]) -------------------
def _plan_or_none(plan):
    return ctypes.byref(plan) if plan is not None else None


def apply_unitary(h: TiledHermitian, u: np.ndarray, targets, plan=None) -> None:
    u = np.ascontiguousarray(u, np.complex128)
    tg, tgp = _u32(targets)
    nat.check(nat.engine().hs_apply_unitary(h.handle, len(tg), _dp(u), tgp, _plan_or_none(plan)), "apply_unitary")


def apply_kraus(h: TiledHermitian, ops: np.ndarray, targets, plan=None) -> None:
    ops = np.ascontiguousarray(ops, np.complex128)
    if ops.ndim == 2:
        ops = ops[None]
    tg, tgp = _u32(targets)
    nat.check(nat.engine().hs_apply_kraus(h.handle, len(tg), ops.shape[0], _dp(ops), tgp, _plan_or_none(plan)),
              "apply_kraus")


def apply_transfer(h: TiledHermitian, s_rowstacked: np.ndarray, targets, plan=None) -> None:
    s = np.ascontiguousarray(s_rowstacked, np.complex128)
    tg, tgp = _u32(targets)
    nat.check(nat.engine().hs_apply_transfer(h.handle, len(tg), _dp(s), tgp, _plan_or_none(plan)), "apply_transfer")


def apply_hadamard(h: TiledHermitian, target: int, plan=None) -> None:
    nat.check(nat.engine().hs_apply_hadamard(h.handle, target, _plan_or_none(plan)), "apply_hadamard")


def apply_diagonal_phase(h: TiledHermitian, target: int, phases, plan=None) -> None:
    p = np.ascontiguousarray(phases, np.complex128)
    nat.check(nat.engine().hs_apply_diagonal_phase(h.handle, target, _dp(p), _plan_or_none(plan)),
              "apply_diagonal_phase")


def apply_permutation(h: TiledHermitian, table, targets, plan=None) -> None:
    t, tp = _u32(table)
    tg, tgp = _u32(targets)
    nat.check(nat.engine().hs_apply_permutation(h.handle, len(tg), tp, tgp, _plan_or_none(plan)),
              "apply_permutation")


def apply_cx_layer(h: TiledHermitian, pairs, plan=None) -> None:
    """CX gates on disjoint (control, target) pairs in one pass (fusion; bit-identical to applying
    native_gate("cnot") on each pair in turn).  Single-GPU states."""
    pairs = [(int(c), int(t)) for c, t in pairs]
    c, cp = _u32([p[0] for p in pairs])
    t, tp = _u32([p[1] for p in pairs])
    nat.check(nat.engine().hs_apply_cx_layer(h.handle, len(pairs), cp, tp, _plan_or_none(plan)), "apply_cx_layer")


def launch_count() -> int:
    return int(nat.engine().hs_launch_count())


def device_count() -> int:
    n = ctypes.c_int()
    nat.check(nat.engine().hs_device_count(ctypes.byref(n)), "device_count")
    return n.value
