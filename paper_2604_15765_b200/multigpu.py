"""Sharding the tiled operator across GPUs.

XOR blocks: with P = 2^p shards and B = G / P tile rows per block, stored tile (ti >= tj) lives on
shard ``(ti // B) ^ (tj // B)``.  Shard 0 holds the P diagonal blocks (triangular), shard s != 0 the
P / 2 rectangular blocks (a, a ^ s) with a > a ^ s.  The layout is balanced to 1 + 1/B, keeps a tile
and its hermitian mirror on the same shard, and P = 1 is exactly the reference's triangle.

* Operations whose targets avoid the top p qubits touch only one shard's tiles: no communication.
* An operation with one target among the top p qubits (bit c) pairs shard s with s ^ 2^c: both sides
  exchange their whole shard (NCCL send/recv over NVLink, one pairwise butterfly step), compute every
  unit they share and store only their own tiles.  With t top targets (mask of their shard bits) the
  group s ^ span(mask) of 2^t shards exchanges all-to-all inside the group the same way (a CX on two
  top qubits: 4 shards).  Every other collective is a scalar sum (expectation values).

``ShardLayout`` is the host-side mirror of the engine's addressing (planning, scatter/gather, tests);
``ShardGroup`` drives P shards from one process (one GPU or several, exchange by device/peer copies);
``DistributedShard`` is one rank of a torch.distributed job (exchange by NCCL inside the engine).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from . import hermsim as H


def _tri(t):
    return t * (t + 1) // 2


class ShardLayout:
    """Tile <-> (shard, local index) mapping of the engine (csrc/engine.cu, shard_index)."""

    def __init__(self, n: int, m: int, nshards: int):
        self.n, self.m, self.P = n, m, nshards
        self.M = 1 << m
        self.G = (1 << n) >> m if n >= m else 1
        if nshards < 1 or nshards & (nshards - 1) or nshards > self.G:
            raise ValueError("shard count must be a power of two <= tiles per grid row")
        self.p = nshards.bit_length() - 1
        self.B = self.G // nshards
        self.top0 = m + (self.G.bit_length() - 1) - self.p  # lowest cross-shard qubit

    def shard_of(self, ti: int, tj: int) -> int:
        return (ti // self.B) ^ (tj // self.B)

    def index(self, ti: int, tj: int, s: int | None = None) -> int:
        """Local tile index of stored tile (ti >= tj) in shard s."""
        s = self.shard_of(ti, tj) if s is None else s
        if self.P == 1:
            return _tri(ti) + tj
        B = self.B
        a, r, c = ti // B, ti % B, tj % B
        if s == 0:
            return a * (B * (B + 1) // 2) + _tri(r) + c
        h = s.bit_length() - 1
        blk = ((a >> (h + 1)) << h) | (a & ((1 << h) - 1))
        return blk * B * B + r * B + c

    def tiles(self, s: int) -> int:
        B, P = self.B, self.P
        return P * (B * (B + 1) // 2) if s == 0 else (P // 2) * B * B

    def count(self, s: int) -> int:
        return self.tiles(s) * self.M * self.M

    def decode(self, s: int, t: int):
        """Local tile index -> (ti, tj)."""
        B = self.B
        if self.P == 1 or s == 0:
            per = B * (B + 1) // 2 if self.P > 1 else None
            a, v = (t // per, t % per) if per else (0, t)
            r = int((np.sqrt(8 * v + 1) - 1) // 2)
            while _tri(r) > v:
                r -= 1
            while _tri(r + 1) <= v:
                r += 1
            return a * B + r, a * B + (v - _tri(r))
        h = s.bit_length() - 1
        blk, v = t // (B * B), t % (B * B)
        a = ((blk >> h) << (h + 1)) | (1 << h) | (blk & ((1 << h) - 1))
        return a * B + v // B, (a ^ s) * B + v % B

    def group_mask(self, targets) -> int:
        """Shard-bit mask of an operation's top targets (0: shard-local)."""
        if self.P == 1:
            return 0
        mask = 0
        for q in targets:
            if q >= self.top0:
                mask |= 1 << (q - self.top0)
        return mask

    def group(self, shard: int, targets) -> list[int]:
        """The shards an operation couples with `shard` (itself first): shard ^ span(mask)."""
        mask = self.group_mask(targets)
        return [shard ^ d for d in range(1 << self.p) if not d & ~mask]

    def partner(self, shard: int, targets) -> int:
        """Partner shard of an operation with one top target (-1: shard-local)."""
        mask = self.group_mask(targets)
        if not mask:
            return -1
        if mask & (mask - 1):
            raise ValueError("operation couples more than two shards: use group()")
        return shard ^ mask

    def tile_slices(self, s: int):
        """[(global tile index, local tile index)] of shard s, in local order."""
        out = []
        for t in range(self.tiles(s)):
            ti, tj = self.decode(s, t)
            out.append((_tri(ti) + tj, t))
        return out

    def scatter(self, full: np.ndarray) -> list[np.ndarray]:
        MM = self.M * self.M
        ft = full.reshape(-1, MM)
        return [np.ascontiguousarray(ft[[g for g, _ in self.tile_slices(s)]].reshape(-1)) for s in range(self.P)]

    def gather(self, parts) -> np.ndarray:
        MM = self.M * self.M
        out = np.empty((self.G * (self.G + 1) // 2, MM), np.complex128)
        for s, part in enumerate(parts):
            pt = part.reshape(-1, MM)
            for g, t in self.tile_slices(s):
                out[g] = pt[t]
        return out.reshape(-1)


def _shard_state(n, m, device, P, s) -> H.TiledHermitian:
    return H.TiledHermitian(n, m, device=device, nshards=P, shard=s)


def op_partner(st: H.TiledHermitian, targets) -> int:
    tg = np.ascontiguousarray(targets, np.uint32)
    out = ctypes.c_int()
    nat.check(nat.engine().hs_op_partner(st.handle, len(tg), tg.ctypes.data_as(nat.c_u32_p), ctypes.byref(out)),
              "op_partner")
    return out.value


def moving_qubits(spec: H.ChannelSpec, targets) -> set:
    """Target qubits whose bit an operation changes: none for a diagonal phase, the permuted bits of
    a permutation (a CX moves only its target), every target otherwise.  Stationary top targets need
    no exchange (the engine skips those remote tiles, hs_apply_monomial)."""
    targets = [int(q) for q in targets]
    if spec.kind == "diagonal_phase":
        return set()
    if spec.kind == "permutation":
        perm = spec.perm
        if perm is not None:
            k, mv = len(targets), 0
            for x, px in enumerate(perm):
                mv |= x ^ int(px)
            return {targets[i] for i in range(k) if mv >> (k - 1 - i) & 1}  # first-listed = MSB
    return set(targets)


def xpattern(spec: H.ChannelSpec) -> bool:
    """A single-qubit channel whose transfer matrix couples only (00, 11) and (01, 10): the two
    shard classes of a cross-shard quad, so it needs no exchange (depolarising,
    amplitude damping, dephasing; the engine's hs_apply_transfer applies the same test)."""
    if spec.k != 1 or spec.kind not in ("generic_kraus",):
        return False
    from .fusion import transfer_rowstacked
    s = transfer_rowstacked(spec.kraus)
    cls = np.array([0, 1, 1, 0])
    return not np.any(s[cls[:, None] != cls[None, :]])


def op_mask(layout: ShardLayout, spec: H.ChannelSpec, targets) -> int:
    """Shard-bit mask of the group an operation must exchange with (0: shard-local)."""
    if xpattern(spec):
        return 0
    return layout.group_mask(sorted(moving_qubits(spec, targets)))


def op_group(st: H.TiledHermitian, targets) -> int:
    tg = np.ascontiguousarray(targets, np.uint32)
    out = ctypes.c_uint32()
    nat.check(nat.engine().hs_op_group(st.handle, len(tg), tg.ctypes.data_as(nat.c_u32_p), ctypes.byref(out)),
              "op_group")
    return out.value


def reduce_partial(a: H.TiledHermitian, b: H.TiledHermitian | None, kind: int) -> float:
    out = ctypes.c_double()
    nat.check(nat.engine().hs_reduce_partial(a.handle, (b or a).handle, kind, ctypes.byref(out)), "reduce")
    return out.value


def _peer_buffers(st: H.TiledHermitian):
    b0, b1 = ctypes.c_void_p(), ctypes.c_void_p()
    nat.check(nat.engine().hs_state_peer_buffers(st.handle, ctypes.byref(b0), ctypes.byref(b1)), "peer buffers")
    return b0, b1


class ShardGroup:
    """P shards of one operator driven from one process (devices: one GPU or a list of GPUs).

    peer=False: a cross-shard op first copies the group members' payloads into exchange slots.
    peer=True: every shard's kernels read the members' current payloads in place (same device or
    peer access) and write out of place; a barrier (all shard streams synchronised) precedes each
    op that touches a top qubit."""

    def __init__(self, n: int, m: int = 5, nshards: int = 2, devices=(0,), peer: bool = False):
        self.layout = ShardLayout(n, m, nshards)
        self.n, self.m, self.P, self.peer = n, m, nshards, peer
        self.shards = [_shard_state(n, m, devices[s % len(devices)], nshards, s) for s in range(nshards)]
        if peer:
            L = nat.engine()
            for st in self.shards:
                nat.check(L.hs_state_peer_enable(st.handle), "peer enable")
            bufs = [_peer_buffers(st) for st in self.shards]
            for a, st in enumerate(self.shards):
                for b, other in enumerate(self.shards):
                    if a != b:
                        nat.check(L.hs_peer_access(st.device, other.device), "peer access")
                        nat.check(L.hs_state_set_peer(st.handle, b, bufs[b][0], bufs[b][1]), "set peer")

    def apply(self, spec: H.ChannelSpec, targets, opts: H.ApplyOptions | None = None):
        """hermsim.apply on every shard; exchanges first when the op crosses shards."""
        opts = opts or H.ApplyOptions(count_subcases=False)
        if self.peer:
            if self.layout.group_mask(targets):  # members read each other: previous ops complete
                for st in self.shards:
                    st.synchronize()
            plans = [H.apply(st, spec, targets, opts) for st in self.shards]
            return plans[0]
        mask = op_mask(self.layout, spec, targets)
        if mask:
            # all exchanges read the pre-op payloads, then every shard updates its own tiles
            for s, st in enumerate(self.shards):
                for peer in [s ^ d for d in range(1, self.P) if not d & ~mask]:
                    nat.check(nat.engine().hs_state_exchange_group_from(st.handle, self.shards[peer].handle, mask),
                              "exchange")
            for st in self.shards:
                st.synchronize()
        plans = [H.apply(st, spec, targets, opts) for st in self.shards]
        return plans[0]

    def apply_sequence(self, ops, opts: H.ApplyOptions | None = None, remap: bool = False, window: int = 24):
        """A sequence of (spec, logical targets); remap=True goes through plan_remap (self.perm holds
        the logical -> physical map; restore_layout() undoes it)."""
        if not hasattr(self, "perm"):
            self.perm = list(range(self.n))
        if not remap:
            return [self.apply(spec, [self.perm[q] for q in tg], opts) for spec, tg in ops]
        actions, _, _ = plan_remap(ops, self.layout, self.perm, window)
        plans = []
        for a in actions:
            if a[0] == "swap":
                self.apply(_swap_spec(), [a[1], a[2]], opts)
            else:
                plans.append(self.apply(a[1], a[2], opts))
        return plans

    def restore_layout(self, opts: H.ApplyOptions | None = None):
        perm = getattr(self, "perm", list(range(self.n)))
        for q in range(self.n):
            while perm[q] != q:
                p = perm[q]
                r = perm.index(q)
                self.apply(_swap_spec(), [p, q], opts)
                perm[q], perm[r] = q, p

    def fill_mixture(self, psi):
        for st in self.shards:
            st.fill_mixture(psi)

    def fill_pauli_sum(self, *strings):
        for st in self.shards:
            st.fill_pauli_sum(*strings)

    def upload_full(self, payload):
        for st, part in zip(self.shards, self.layout.scatter(payload)):
            st.upload(part)

    def download_full(self) -> np.ndarray:
        return self.layout.gather([st.download() for st in self.shards])

    def expectation(self, obs: "ShardGroup") -> float:
        return float(sum(reduce_partial(o, r, 0) for r, o in zip(self.shards, obs.shards)))

    def trace(self) -> float:
        return float(sum(reduce_partial(st, None, 2) for st in self.shards))

    def synchronize(self):
        for st in self.shards:
            st.synchronize()

    def free(self):
        for st in self.shards:
            st.free()


class EngineBackend:
    """What DistributedShard asks of the device side: the CUDA engine (the product path).  The CPU
    tests substitute an emulator with the same methods (tests/shard_emu.py), so the rank protocol --
    ownership, exchange plan, barriers, remapping, reductions -- runs unchanged under gloo."""

    def state(self, n, m, device, nshards, shard):
        return _shard_state(n, m, device, nshards, shard)

    def connect_peer(self, sh: "DistributedShard"):
        import torch.distributed as dist
        L = nat.engine()
        nat.check(L.hs_state_peer_enable(sh.state.handle), "peer enable")
        hd = (ctypes.c_char * 128)()
        nat.check(L.hs_ipc_handles(sh.state.handle, hd), "ipc handles")
        allh = [None] * sh.world
        dist.all_gather_object(allh, (bytes(hd), sh.device))
        for r, (h, dev) in enumerate(allh):
            if r == sh.rank:
                continue
            if dev != sh.device:
                nat.check(L.hs_peer_access(sh.device, dev), "peer access")
            ptrs = []
            for half in (h[:64], h[64:]):
                p = ctypes.c_void_p()
                nat.check(L.hs_ipc_open((ctypes.c_char * 64).from_buffer_copy(half), sh.device, ctypes.byref(p)),
                          "ipc open")
                ptrs.append(p)
                sh._opened.append(p)
            nat.check(L.hs_state_set_peer(sh.state.handle, r, ptrs[0], ptrs[1]), "set peer")

    def connect_nccl(self, sh: "DistributedShard"):
        import torch.distributed as dist
        uid = (ctypes.c_char * 128)()
        if sh.rank == 0:
            nat.check(nat.engine().hs_nccl_unique_id(uid), "nccl id")
        obj = [bytes(uid) if sh.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        buf = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        nat.check(nat.engine().hs_state_comm_init(sh.state.handle, buf, sh.world, sh.rank), "comm init")

    def exchange(self, sh: "DistributedShard", mask: int):
        nat.check(nat.engine().hs_state_exchange_group(sh.state.handle, mask), "exchange")

    def apply(self, sh: "DistributedShard", spec, targets, opts):
        return H.apply(sh.state, spec, targets, opts)

    def synchronize(self, sh: "DistributedShard"):
        sh.state.synchronize()

    def reduce_partial(self, a, b, kind: int) -> float:
        return reduce_partial(a, b, kind)

    def close(self, sh: "DistributedShard"):
        if sh.peer:
            sh.state.synchronize()
            for p in sh._opened:
                nat.engine().hs_ipc_close(p, sh.device)
            sh._opened = []


SWAP = None  # hermsim SWAP spec, built on first use


def _swap_spec():
    global SWAP
    if SWAP is None:
        SWAP = H.native_gate("swap")
    return SWAP


def plan_remap(ops, layout: ShardLayout, perm: list, window: int = 24):
    """Qubit remapping for sharded runs: rewrite a sequence of (spec, logical
    targets) into physical actions, swapping a top (cross-shard) qubit with a low one when that
    saves exchanges.  perm[logical] = physical qubit (updated in place).

    Before an operation that needs an exchange, for each top physical qubit it moves: try swapping
    it with every low physical qubit not among the operation's targets, and take the swap (one SWAP
    = one exchange) when the exchanges of the next `window` operations drop by more than one.
    Returns [("swap", pa, pb) | ("op", spec, physical targets)] and the number of exchanges without /
    with remapping (swaps included)."""
    top0 = layout.top0
    cache = {}

    def needs(spec, logical, mp):
        key = id(spec)
        if key not in cache:
            cache[key] = (xpattern(spec), spec)
        if cache[key][0]:
            return 0
        return layout.group_mask(sorted(mp[q] for q in moving_qubits(spec, logical)))

    def cost(horizon, mp):
        return sum(1 for sp, t2 in horizon if needs(sp, t2, mp))

    ident = list(range(len(perm)))
    out, plain, remapped = [], 0, 0
    for i, (spec, tg) in enumerate(ops):
        plain += 1 if needs(spec, tg, ident) else 0
        mask = needs(spec, tg, perm)
        if mask:
            horizon = ops[i:i + window]
            for q in tg:
                pq = perm[q]
                if pq < top0 or not (mask >> (pq - top0) & 1):
                    continue
                base = cost(horizon, perm)
                best, best_p = base - 1, None  # a swap must save more than its own exchange
                for p in range(top0):
                    r = perm.index(p)
                    if r in tg:
                        continue
                    trial = list(perm)
                    trial[q], trial[r] = p, pq
                    c = cost(horizon, trial)
                    if c < best:
                        best, best_p = c, p
                if best_p is not None:
                    r = perm.index(best_p)
                    out.append(("swap", pq, best_p))
                    remapped += 1
                    perm[q], perm[r] = best_p, pq
                    mask = needs(spec, tg, perm)
        remapped += 1 if mask else 0
        out.append(("op", spec, [perm[q] for q in tg]))
    return out, plain, remapped


class DistributedShard:
    """This rank's shard of an operator sharded over a torch.distributed job (rank == shard).

    peer=False: the cross-shard exchange runs inside the engine over NCCL on the state's stream.
    peer=True: the ranks map each other's two payload buffers (CUDA IPC; peer access over NVLink) and
    a cross-shard op's kernels read the group members' tiles in place -- the collective is fused
    into the op; a barrier precedes each op that touches a top qubit.
    remap=True: operations go through qubit remapping (plan_remap): logical targets are mapped to
    physical qubits, and top qubits that keep needing exchanges are swapped down first.
    backend: the device side (EngineBackend; the CPU tests pass an emulator)."""

    def __init__(self, n: int, m: int = 5, device: int | None = None, peer: bool = False, remap: bool = False,
                 backend=None):
        import torch.distributed as dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.layout = ShardLayout(n, m, self.world)
        self.n, self.m = n, m
        self.device = self.rank if device is None else device
        self.backend = backend or EngineBackend()
        self.state = self.backend.state(n, m, self.device, self.world, self.rank)
        self.peer = peer
        self.remap = remap
        self.perm = list(range(n))  # logical -> physical qubit
        self.exchanges = 0
        self._opened = []
        if peer:
            self.backend.connect_peer(self)
        else:
            self.backend.connect_nccl(self)

    def _apply_physical(self, spec, targets, opts):
        if self.peer:
            if self.layout.group_mask(targets):  # members read each other: previous ops complete
                import torch.distributed as dist
                self.backend.synchronize(self)
                dist.barrier()
                self.exchanges += 1
            return self.backend.apply(self, spec, targets, opts)
        mask = op_mask(self.layout, spec, targets)
        if mask:
            self.backend.exchange(self, mask)
            self.exchanges += 1
        return self.backend.apply(self, spec, targets, opts)

    def apply(self, spec: H.ChannelSpec, targets, opts: H.ApplyOptions | None = None):
        opts = opts or H.ApplyOptions(count_subcases=False)
        if not self.remap:
            return self._apply_physical(spec, list(targets), opts)
        return self._apply_physical(spec, [self.perm[q] for q in targets], opts)

    def apply_sequence(self, ops, opts: H.ApplyOptions | None = None, window: int = 24):
        """A sequence of (spec, logical targets); with remap=True through plan_remap (swaps inserted)."""
        opts = opts or H.ApplyOptions(count_subcases=False)
        if not self.remap:
            return [self._apply_physical(spec, list(tg), opts) for spec, tg in ops]
        actions, _, _ = plan_remap(ops, self.layout, self.perm, window)
        plans = []
        for a in actions:
            if a[0] == "swap":
                self._apply_physical(_swap_spec(), [a[1], a[2]], opts)
            else:
                plans.append(self._apply_physical(a[1], a[2], opts))
        return plans

    def restore_layout(self, opts: H.ApplyOptions | None = None):
        """Swap qubits back until logical == physical (the payload is then the unremapped one)."""
        opts = opts or H.ApplyOptions(count_subcases=False)
        for q in range(self.n):
            while self.perm[q] != q:
                p = self.perm[q]
                r = self.perm.index(q)  # the logical qubit sitting on physical q
                self._apply_physical(_swap_spec(), [p, q], opts)
                self.perm[q], self.perm[r] = q, p

    def close(self):
        """Unmaps the peers' buffers (peer mode); the state itself is freed with the object."""
        self.backend.close(self)

    def reduce(self, other: "DistributedShard | None", kind: int) -> float:
        """Sum over shards of the partial (deterministic: gathered, summed in rank order)."""
        import torch.distributed as dist
        part = self.backend.reduce_partial(self.state, other.state if other else None, kind)
        parts = [None] * self.world
        dist.all_gather_object(parts, part)
        return float(sum(parts))
