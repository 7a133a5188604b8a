"""CPU emulation of the engine's per-shard unit kernel (TEST INFRASTRUCTURE): numpy on whole tiles,
mirroring csrc/engine.cu's rules -- enumerate units, read logical tiles from the local payload or the
exchange buffer (adjoint tiles conjugate-transposed), compute every component, store only tiles this
shard owns (and, on diagonal units, only R >= C).  Used by the gloo multi-process test to check the
sharding plan (ownership, partner, exchange) without a GPU."""
import numpy as np


def _ins(x, bit, pos):
    return (((x >> pos) << 1 | bit) << pos) | (x & ((1 << pos) - 1))


def apply_k1(layout, s, local, recv, srow, a):
    """k = 1 transfer-matrix channel (srow: row-stacked 4x4) on qubit a, shard s, in place on local."""
    M, m = layout.M, layout.m
    loc = local.reshape(-1, M, M)
    rcv = None if recv is None else recv.reshape(-1, M, M)
    if a < m:  # intra: every local tile independently
        bit = 1 << a
        base = [r for r in range(M) if not r & bit]
        for t in range(loc.shape[0]):
            T = loc[t]
            for r0 in base:
                r1 = r0 + bit
                for c0 in base:
                    c1 = c0 + bit
                    v = np.array([T[r0, c0], T[r0, c1], T[r1, c0], T[r1, c1]])
                    T[r0, c0], T[r0, c1], T[r1, c0], T[r1, c1] = srow @ v
        return
    ap = a - m
    nb = layout.G // 2
    for tbi in range(nb):
        for tbj in range(tbi + 1):
            tr = [_ins(tbi, R, ap) for R in range(2)]
            tc = [_ins(tbj, C, ap) for C in range(2)]
            owners = {}
            for R in range(2):
                for C in range(2):
                    hi, lo = max(tr[R], tc[C]), min(tr[R], tc[C])
                    owners[(R, C)] = (layout.shard_of(hi, lo), hi, lo, tr[R] < tc[C])
            if all(o[0] != s for o in owners.values()):
                continue
            tiles = {}
            for (R, C), (own, hi, lo, adj) in owners.items():
                src = loc if own == s else rcv
                T = src[layout.index(hi, lo, own)]
                tiles[(R, C)] = T.conj().T if adj else T
            v = np.stack([tiles[(0, 0)], tiles[(0, 1)], tiles[(1, 0)], tiles[(1, 1)]])
            w = np.tensordot(srow, v, axes=(1, 0))
            out = {(0, 0): w[0], (0, 1): w[1], (1, 0): w[2], (1, 1): w[3]}
            for (R, C), (own, hi, lo, adj) in owners.items():
                if own != s or (tbi == tbj and R < C):
                    continue
                loc[layout.index(hi, lo, own)] = out[(R, C)].conj().T if adj else out[(R, C)]
