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


class DistributedShard:
    """This rank's shard of an operator sharded over a torch.distributed job (rank == shard).

    peer=False: the cross-shard exchange runs inside the engine over NCCL on the state's stream.
    peer=True: the ranks map each other's two payload buffers (CUDA IPC; peer access over NVLink) and
    a cross-shard op's kernels read the group members' tiles in place -- the collective is fused
    into the op; a barrier precedes each op that touches a top qubit."""

    def __init__(self, n: int, m: int = 5, device: int | None = None, peer: bool = False):
        import torch.distributed as dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.layout = ShardLayout(n, m, self.world)
        self.device = self.rank if device is None else device
        self.state = _shard_state(n, m, self.device, self.world, self.rank)
        self.peer = peer
        self._opened = []
        if peer:
            L = nat.engine()
            nat.check(L.hs_state_peer_enable(self.state.handle), "peer enable")
            hd = (ctypes.c_char * 128)()
            nat.check(L.hs_ipc_handles(self.state.handle, hd), "ipc handles")
            allh = [None] * self.world
            dist.all_gather_object(allh, (bytes(hd), self.device))
            for r, (h, dev) in enumerate(allh):
                if r == self.rank:
                    continue
                if dev != self.device:
                    nat.check(L.hs_peer_access(self.device, dev), "peer access")
                ptrs = []
                for half in (h[:64], h[64:]):
                    p = ctypes.c_void_p()
                    nat.check(L.hs_ipc_open((ctypes.c_char * 64).from_buffer_copy(half), self.device,
                                            ctypes.byref(p)), "ipc open")
                    ptrs.append(p)
                    self._opened.append(p)
                nat.check(L.hs_state_set_peer(self.state.handle, r, ptrs[0], ptrs[1]), "set peer")
            return
        uid = (ctypes.c_char * 128)()
        if self.rank == 0:
            nat.check(nat.engine().hs_nccl_unique_id(uid), "nccl id")
        obj = [bytes(uid) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        buf = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        nat.check(nat.engine().hs_state_comm_init(self.state.handle, buf, self.world, self.rank), "comm init")

    def apply(self, spec: H.ChannelSpec, targets, opts: H.ApplyOptions | None = None):
        opts = opts or H.ApplyOptions(count_subcases=False)
        if self.peer:
            if self.layout.group_mask(targets):  # members read each other: previous ops complete
                import torch.distributed as dist
                self.state.synchronize()
                dist.barrier()
            return H.apply(self.state, spec, targets, opts)
        mask = op_mask(self.layout, spec, targets)
        if mask:
            nat.check(nat.engine().hs_state_exchange_group(self.state.handle, mask), "exchange")
        return H.apply(self.state, spec, targets, opts)

    def close(self):
        """Unmaps the peers' buffers (peer mode); the state itself is freed with the object."""
        if self.peer:
            self.state.synchronize()
            for p in self._opened:
                nat.engine().hs_ipc_close(p, self.device)
            self._opened = []

    def reduce(self, other: "DistributedShard | None", kind: int) -> float:
        """Sum over shards of the partial (deterministic: gathered, summed in rank order)."""
        import torch.distributed as dist
        part = reduce_partial(self.state, other.state if other else None, kind)
        parts = [None] * self.world
        dist.all_gather_object(parts, part)
        return float(sum(parts))
