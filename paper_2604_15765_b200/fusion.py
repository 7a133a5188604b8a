"""Operation fusion: fewer HBM passes for the same operation sequence.

The reference applies one operation per pass over the tiled triangle (`hermsim::apply`,
kernels.cpp:510-549). ``apply_sequence`` gives the same result for a whole sequence with fewer passes:

* a run of consecutive single-qubit operations is regrouped per qubit (single-qubit channels on
  different qubits commute);
* the operations of each qubit form a chain of steps, each in its cheapest form (Hadamard butterfly,
  diagonal phase, real (00,11)/(01,10) transfer as for depolarising / amplitude damping, or a general
  transfer matrix); neighbours are composed into one transfer matrix S = S_last ... S_first
  (row-stacked, the engine's `TransferQuad` order, kernels.cpp:66-77) only where that is cheaper;
* the chains of all in-tile qubits (< m) of the run go into ONE pass (`hs_apply_program`): the
  staged tiles are transformed qubit after qubit in shared memory, each qubit's chain running on a
  quad in registers (one shared-memory round trip per qubit);
* the chains of up to three grid qubits share one pass (`hs_apply_grid_program`: the units of those
  grid bits are gathered and each qubit's chain applied per quad; m = 5); a lone grid qubit's chain
  is composed into one transfer matrix; without grid programs, two unitary grid steps share a pass
  as U_a (x) U_b (tensor-core gather);
* any other operation (k >= 2) ends the run; consecutive multi-qubit unitaries on the same qubit
  set (C1's CX then Haar U on each ordered pair) are composed into one unitary U2 U1 (the second
  re-indexed to the first's target order, first-listed target = most significant bit,
  channel.cpp:209-216) and applied in one pass;
* consecutive CX gates on disjoint qubit pairs (C4's matchings) run as one in-place permutation
  pass (`hs_apply_cx_layer`, bit-identical to one CX after the other).

The result equals applying the sequence one operation at a time up to floating-point rounding
(the composition reorders products); ``tests/test_gpu_fusion.py`` checks it at 1e-12 * ||rho||_F.
Throughput with fusion is reported separately from the per-operation metric (bench.py --fuse).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import hermsim as H


def transfer_rowstacked(kraus: np.ndarray) -> np.ndarray:
    """Row-stacked 4 x 4 transfer matrix of a single-qubit Kraus set: w[r*2+c] = sum S v[r'*2+c'],
    S[(r, c), (r', c')] = sum_a K_a[r, r'] conj(K_a[c, c']) (H' = sum_a K_a H K_a^dagger)."""
    k = np.asarray(kraus, np.complex128).reshape(-1, 2, 2)
    s = np.einsum("arp,acq->rcpq", k, k.conj())
    return s.reshape(4, 4)


@dataclass
class Step:
    qubit: int
    s: np.ndarray            # row-stacked 4 x 4
    lone_h: bool = False     # exactly one native Hadamard
    count: int = 1           # operations composed into this step
    u: np.ndarray | None = None  # 2 x 2 unitary when every composed operation is one (S = conj(U) (x) U)


@dataclass
class Plan:
    """Launch list of a fused sequence: ("program", [Step]) | ("step", Step) | ("op", spec, targets)."""
    items: list = field(default_factory=list)
    ops: int = 0

    @property
    def launches(self) -> int:
        return len(self.items)


def _single_qubit_s(spec: H.ChannelSpec) -> np.ndarray:
    return transfer_rowstacked(spec.kraus)


def _unitary_of(spec: H.ChannelSpec) -> np.ndarray | None:
    k = spec.kraus
    if k.shape[0] != 1:
        return None
    u = k[0]
    return u if np.allclose(u @ u.conj().T, np.eye(2), atol=1e-14) else None


def reorder_targets(u: np.ndarray, src: list, dst: list) -> np.ndarray:
    """The k-qubit operator u written for targets `src` (first listed = most significant bit),
    re-indexed for the same qubits listed as `dst`."""
    k = len(src)
    perm = [src.index(q) for q in dst]
    t = np.asarray(u).reshape((2,) * (2 * k))
    return t.transpose(perm + [k + p for p in perm]).reshape(1 << k, 1 << k)


def _unitary_k(spec: H.ChannelSpec) -> np.ndarray | None:
    if spec.nops != 1:
        return None
    u = spec.kraus[0]
    return u if np.allclose(u @ u.conj().T, np.eye(u.shape[0]), atol=1e-13) else None


def _is_cx(spec: H.ChannelSpec) -> bool:
    return spec.kind == "permutation" and spec.k == 2 and spec.name == "cnot"


def _compose(chain: list) -> Step:
    """One step equal to a qubit's chain applied in order (S = S_last ... S_first)."""
    st = chain[0]
    for x in chain[1:]:
        uu = x.u @ st.u if (x.u is not None and st.u is not None) else None
        st = Step(st.qubit, x.s @ st.s, False, st.count + x.count, uu)
    return st


def plan_sequence(ops, n: int, m: int = 5, pair_unitaries: bool = True, grid_groups: int = 3,
                  compose_multi: bool = True, cx_layers: bool = True) -> Plan:
    """ops: iterable of (ChannelSpec, targets)."""
    plan = Plan()
    cx_pend: list = []  # consecutive CX on disjoint pairs: [(spec, [control, target])]

    def emit_cx():
        if len(cx_pend) >= 2:
            plan.items.append(("cxlayer", [tuple(tg) for _, tg in cx_pend]))
        else:
            for spec, tg in cx_pend:
                plan.items.append(("op", spec, tg))
        cx_pend.clear()
    edge = min(m, n)  # in-tile qubits
    order: list[int] = []
    # per qubit: a chain of steps applied in order.  A program runs a qubit's chain on each quad in
    # registers (one shared-memory round trip per qubit), so steps are composed only where the
    # composition's arithmetic is cheaper than the chain's (_KIND_COST)
    chains: dict[int, list[Step]] = {}

    def flush():
        intile = [x for q in order if q < edge for x in chains[q]]
        for i in range(0, len(intile), 16):
            plan.items.append(("program", intile[i:i + 16]))
        grid = [q for q in order if q >= edge]
        if grid_groups > 1 and m == 5:
            # grid qubits three (two) at a time in one gathered pass (hs_apply_grid_program), each
            # with its chain; at most 16 steps per pass
            i = 0
            while i < len(grid):
                grp = grid[i:i + grid_groups]
                while len(grp) > 1 and sum(len(chains[q]) for q in grp) > 16:
                    grp = grp[:-1]
                if len(grp) == 1:
                    plan.items.append(("step", _compose(chains[grp[0]])))
                else:
                    plan.items.append(("gprogram", [x for q in grp for x in chains[q]]))
                i += len(grp)
            chains.clear()
            order.clear()
            return
        # grid qubits: two unitary steps share one pass as the 2-qubit unitary U_a (x) U_b (the
        # tensor-core gather, k = 2 on two grid bits); others are one pass each
        pend = None
        for q in grid:
            st = _compose(chains[q])
            if pair_unitaries and st.u is not None:
                if pend is None:
                    pend = st
                    continue
                u2 = np.kron(pend.u, st.u)  # first-listed target (pend) is the most significant bit
                plan.items.append(("op", H.make_generic("fused_u2", u2), [pend.qubit, st.qubit]))
                pend = None
                continue
            plan.items.append(("step", st))
        if pend is not None:
            plan.items.append(("step", pend))
        chains.clear()
        order.clear()

    for spec, targets in ops:
        targets = list(targets)
        plan.ops += 1
        if cx_layers and _is_cx(spec) and len(targets) == 2:
            flush()
            if any(q in (c, t) for _, (c, t) in cx_pend for q in targets):
                emit_cx()
            cx_pend.append((spec, targets))
            continue
        emit_cx()
        if spec.k != 1 or len(targets) != 1:
            flush()
            last = plan.items[-1] if plan.items else None
            if (compose_multi and last is not None and last[0] == "op" and len(last) == 3
                    and sorted(last[2]) == sorted(targets)):
                u1, u2 = _unitary_k(last[1]), _unitary_k(spec)
                if u1 is not None and u2 is not None:
                    u = reorder_targets(u2, targets, last[2]) @ u1
                    plan.items[-1] = ("op", H.make_generic("fused_u", u), last[2])
                    continue
            plan.items.append(("op", spec, targets))
            continue
        q = int(targets[0])
        step = Step(q, _single_qubit_s(spec), spec.kind == "hadamard", 1, _unitary_of(spec))
        ch = chains.setdefault(q, [])
        if not ch:
            order.append(q)
        else:
            comp = _compose([ch[-1], step])
            if _KIND_COST[_kind(comp)] <= _KIND_COST[_kind(ch[-1])] + _KIND_COST[_kind(step)]:
                ch.pop()
                step = comp
        ch.append(step)
    emit_cx()
    flush()
    return plan


_XPAT = np.zeros((4, 4), bool)
for _r, _c in ((0, 0), (0, 3), (3, 0), (3, 3), (1, 1), (1, 2), (2, 1), (2, 2)):
    _XPAT[_r, _c] = True


def _kind(step: Step) -> int:
    """Cheapest kernel form of a step: 1 Hadamard, 2 diagonal, 3 real (00,11)/(01,10), 4 real (00,11)
    block with a complex diagonal on (01,10) (kind 3 channels composed with Rz / phase gates),
    0 general."""
    if step.lone_h:
        return 1
    s = step.s
    if not np.any(s - np.diag(np.diag(s))):
        return 2
    if not np.any(s.imag) and not np.any(s[~_XPAT]):
        return 3
    if (not np.any(s[~_XPAT]) and s[1, 2] == 0 and s[2, 1] == 0
            and not np.any(s[np.ix_([0, 3], [0, 3])].imag)):
        return 4
    return 0


# relative arithmetic of a step per quad (FP64): Hadamard butterfly (adds), diagonal (4 complex
# products), real (00,11)/(01,10) transfer (6 real x complex products) or its composition with a
# diagonal (kind 4, the same count), general 4 x 4 transfer (16 complex FMA); a qubit's chain shares
# one shared-memory round trip, so only this counts
_KIND_COST = {1: 0.5, 2: 1.0, 3: 1.0, 4: 1.0, 0: 4.0}


def _program_args(steps):
    """(kinds, bits, coefficients) of a program's steps.  A Hadamard that follows a coefficient
    step on the same qubit runs as the bare butterfly (kind 5) with its factor 1/2 folded into that
    step's coefficients -- a power of two, so the results are bit for bit the same."""
    kinds = [_kind(x) for x in steps]
    s = np.stack([x.s for x in steps]).astype(np.complex128)
    for i in range(1, len(steps)):
        if kinds[i] == 1 and steps[i - 1].qubit == steps[i].qubit and kinds[i - 1] in (0, 2, 3, 4):
            s[i - 1] = s[i - 1] * 0.5
            kinds[i] = 5
    return (np.array(kinds, np.int32), np.array([x.qubit for x in steps], np.uint32), np.ascontiguousarray(s))


def execute(st: H.TiledHermitian, plan: Plan, opts: H.ApplyOptions | None = None) -> int:
    """Runs a plan on a state; returns the number of passes (launch groups) issued."""
    opts = opts or H.ApplyOptions(count_subcases=False)
    L = nat.engine()
    for item in plan.items:
        if item[0] == "program":
            kinds, bits, s = _program_args(item[1])
            steps = item[1]
            nat.check(L.hs_apply_program(st.handle, len(steps), kinds.ctypes.data_as(nat.c_i32_p),
                                         bits.ctypes.data_as(nat.c_u32_p), s.ctypes.data_as(nat.c_double_p), None),
                      "apply_program")
        elif item[0] == "gprogram":
            kinds, bits, s = _program_args(item[1])
            steps = item[1]
            nat.check(L.hs_apply_grid_program(st.handle, len(steps), kinds.ctypes.data_as(nat.c_i32_p),
                                              bits.ctypes.data_as(nat.c_u32_p), s.ctypes.data_as(nat.c_double_p),
                                              None), "apply_grid_program")
        elif item[0] == "cxlayer":
            H.apply_cx_layer(st, item[1])
        elif item[0] == "step":
            x = item[1]
            if x.lone_h:
                H.apply_hadamard(st, x.qubit)
            else:
                H.apply_transfer(st, np.ascontiguousarray(x.s), [x.qubit])
        else:
            H.apply(st, item[1], item[2], opts)
    return plan.launches


def apply_sequence(st: H.TiledHermitian, ops, opts: H.ApplyOptions | None = None) -> Plan:
    """Fused equivalent of `for spec, tg in ops: hermsim.apply(st, spec, tg)`."""
    plan = plan_sequence(ops, st.qubits(), st.tile_exp())
    execute(st, plan, opts)
    return plan


_ = ctypes
