"""CPU emulation of the device side of a sharded run (TEST INFRASTRUCTURE): stands in for
multigpu.EngineBackend so that the real multigpu.DistributedShard -- ownership, exchange plan
(op_mask), barriers, qubit remapping, reductions -- runs on CPU ranks over torch.distributed gloo.

Each rank holds only its XOR-block shard (numpy).  An exchange sends the whole shard to every other
member of the operation's group and receives theirs (gloo isend / irecv: the NCCL send / recv of the
engine).  Applying an operation rebuilds a dense matrix from the own and the received tiles --
every other element is NaN -- applies the channel block-locally (exactly-zero coefficients skipped,
so a tile that is not read never contaminates one that is) and keeps the own tiles, which must be
NaN-free: the exchanged group suffices.  An exchange licenses one operation, as in the engine."""
import numpy as np


def apply_kraus_dense(rho: np.ndarray, n: int, kraus: np.ndarray, targets) -> np.ndarray:
    """sum_a K rho K^dagger with K acting on `targets` (first-listed = MSB), block-local."""
    k, d = len(targets), 1 << len(targets)
    t = rho.reshape([2] * (2 * n))
    rows = [n - 1 - q for q in targets]
    cols = [2 * n - 1 - q for q in targets]

    def side(x, axes, K):
        x = np.moveaxis(x, axes, list(range(k))).reshape((d,) + x.shape[k:])
        y = np.zeros_like(x)
        for r in range(d):
            for c in range(d):
                if K[r, c] != 0:
                    y[r] = y[r] + K[r, c] * x[c]
        return np.moveaxis(y.reshape([2] * k + list(x.shape[1:])), list(range(k)), axes)

    out = np.zeros_like(t)
    for K in kraus:
        out = out + side(side(t, rows, K), cols, K.conj())
    return out.reshape(rho.shape)


def tiles_to_dense(layout, parts: dict, n: int, m: int) -> np.ndarray:
    """Dense N x N matrix from the tiles of the given shards (hermitian mirrors filled), NaN elsewhere."""
    N, M = 1 << n, 1 << m
    d = np.full((N, N), np.nan + 1j * np.nan, np.complex128)
    for s, payload in parts.items():
        pt = payload.reshape(-1, M, M)
        for t in range(layout.tiles(s)):
            ti, tj = layout.decode(s, t)
            d[ti * M:(ti + 1) * M, tj * M:(tj + 1) * M] = pt[t]
            if ti != tj:
                d[tj * M:(tj + 1) * M, ti * M:(ti + 1) * M] = pt[t].conj().T
    return d


def own_tiles(layout, s: int, d: np.ndarray, m: int) -> np.ndarray:
    M = 1 << m
    out = np.empty((layout.tiles(s), M, M), np.complex128)
    for t in range(layout.tiles(s)):
        ti, tj = layout.decode(s, t)
        out[t] = d[ti * M:(ti + 1) * M, tj * M:(tj + 1) * M]
    return out.reshape(-1)


class EmuState:
    def __init__(self, layout, shard):
        self.layout, self.shard = layout, shard
        self.payload = np.zeros(layout.count(shard), np.complex128)
        self.recv = {}      # member shard -> its payload (last exchange)
        self.license = 0    # shard-bit mask of the last exchange (single use)

    def element_count(self):
        return self.payload.size

    def download(self):
        return self.payload.copy()

    def upload(self, p):
        self.payload[:] = p


class EmuPlan:
    def __init__(self, mask):
        self.mask = mask
        self.touched_bytes = 0


class EmuBackend:
    """multigpu.EngineBackend's methods on numpy shards and gloo point-to-point messages."""

    def __init__(self):
        self.applied = 0

    def state(self, n, m, device, nshards, shard):
        from paper_2604_15765_b200.multigpu import ShardLayout
        return EmuState(ShardLayout(n, m, nshards), shard)

    def connect_peer(self, sh):
        pass

    def connect_nccl(self, sh):
        pass

    def _swap_with_group(self, sh, mask):
        import torch
        import torch.distributed as dist
        st = sh.state
        members = [sh.rank ^ d for d in range(1, sh.world) if not d & ~mask]
        send = torch.from_numpy(st.payload.view(np.float64).copy())
        bufs, reqs = {}, []
        for p in members:
            bufs[p] = torch.from_numpy(np.zeros(st.layout.count(p), np.complex128).view(np.float64))
        for p in members:  # lower rank sends first: no deadlock with blocking-free isend / irecv
            reqs.append(dist.isend(send, p))
            reqs.append(dist.irecv(bufs[p], p))
        for r in reqs:
            r.wait()
        st.recv = {p: b.numpy().view(np.complex128) for p, b in bufs.items()}
        st.license = mask

    def exchange(self, sh, mask):
        self._swap_with_group(sh, mask)

    def apply(self, sh, spec, targets, opts):
        from paper_2604_15765_b200.multigpu import op_mask
        st = sh.state
        need = op_mask(st.layout, spec, targets)
        if sh.peer and need:  # the kernels would read the members' buffers in place
            self._swap_with_group(sh, need)
        if need and (need & ~st.license):
            raise RuntimeError("cross-shard operation without the group's payloads")
        parts = {st.shard: st.payload}
        if need:
            parts.update({p: v for p, v in st.recv.items() if not (p ^ st.shard) & ~need})
        n, m = st.layout.n, st.layout.m
        dense = tiles_to_dense(st.layout, parts, n, m)
        dense = apply_kraus_dense(dense, n, spec.kraus, list(targets))
        mine = own_tiles(st.layout, st.shard, dense, m)
        if np.isnan(mine).any():
            raise AssertionError(f"{spec.name} {list(targets)}: an unexchanged tile reached shard {st.shard}")
        st.payload[:] = mine
        st.license = 0
        st.recv = {}
        self.applied += 1
        return EmuPlan(need)

    def synchronize(self, sh):
        pass

    def reduce_partial(self, a, b, kind):
        """kind 0: tr(a b) part, 1: squared Frobenius part, 2: trace part (csrc reduce_kernel)."""
        b = b or a
        L, M = a.layout, a.layout.M
        pa, pb = a.payload.reshape(-1, M, M), b.payload.reshape(-1, M, M)
        tot = 0.0
        for t in range(L.tiles(a.shard)):
            ti, tj = L.decode(a.shard, t)
            if kind == 2:
                tot += float(np.trace(pa[t]).real) if ti == tj else 0.0
                continue
            v = float(np.sum(pa[t].real * pb[t].real + pa[t].imag * pb[t].imag))
            tot += v if ti == tj else 2 * v
        return tot

    def close(self, sh):
        pass
