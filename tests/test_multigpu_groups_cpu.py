"""Group exchange protocol of the sharded path on CPU (TEST INFRASTRUCTURE: numpy + torch.distributed
gloo, 4 ranks): each rank holds only its XOR-block shard, exchanges with the group that
multigpu.op_mask names (all-to-all inside the group, nothing for stationary top targets), rebuilds
the coupled blocks from its own and the received tiles -- every other tile is NaN -- applies the
operation block-locally and keeps its own tiles.  No NaN may reach a rank's own tiles (the group's
data suffices) and the gathered result must equal applying the sequence to the whole matrix."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def apply_kraus(rho: np.ndarray, n: int, kraus: np.ndarray, targets) -> np.ndarray:
    """sum_a K rho K^dagger with K acting on `targets` (first-listed = MSB), block-local: values
    mix only inside the 2^k x 2^k blocks the operation couples, and exactly-zero coefficients are
    skipped (a permutation moves elements; it never multiplies a tile it does not read by 0)."""
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


def _tiles_to_dense(layout, parts: dict, n: int, m: int) -> np.ndarray:
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


def _own_tiles(layout, s: int, d: np.ndarray, m: int) -> np.ndarray:
    M = 1 << m
    out = np.empty((layout.tiles(s), M, M), np.complex128)
    for t in range(layout.tiles(s)):
        ti, tj = layout.decode(s, t)
        out[t] = d[ti * M:(ti + 1) * M, tj * M:(tj + 1) * M]
    return out.reshape(-1)


def _worker(rank, world, port, n, m, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import ShardLayout, op_mask
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    L = ShardLayout(n, m, world)
    full = HS.rho_payload(n, HS.rank_psi(n, 7, 4), m)
    mine = L.scatter(full)[rank].copy()
    top, exchanged = n - 1, []
    for spec, tg in _ops(H, HS, top):
        mask = op_mask(L, spec, tg)
        exchanged.append(mask)
        parts = {rank: mine}
        peers = [rank ^ d for d in range(1, world) if not d & ~mask] if mask else []
        for peer in peers:  # all-to-all inside the group (the engine's grouped NCCL send/recv)
            buf = torch.zeros(2 * L.count(peer), dtype=torch.float64)
            send = torch.from_numpy(mine.view(np.float64).copy())
            reqs = [dist.isend(send, peer), dist.irecv(buf, peer)] if rank < peer else \
                   [dist.irecv(buf, peer), dist.isend(send, peer)]
            for r in reqs:
                r.wait()
            parts[peer] = buf.numpy().view(np.complex128).copy()
        d = _tiles_to_dense(L, parts, n, m)
        d = apply_kraus(d, n, spec.kraus, tg)
        mine = _own_tiles(L, rank, d, m)
        assert not np.isnan(mine).any(), (spec.name, tg, mask)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        q.put((L.gather(gathered), exchanged))
    dist.destroy_process_group()


def _ops(H, HS, top):
    u2 = HS.haar(2, 31)
    u3 = HS.haar(3, 32)
    return [
        (H.native_gate("cnot"), [top, top - 1]),      # target top-1 moves: 2-shard group
        (H.native_gate("swap"), [top, top - 1]),      # both move: 4-shard group
        (H.make_generic("u2", u2), [top - 1, top]),   # 4-shard group
        (H.depolarising(0.1), [top]),
        (H.make_generic("u3", u3), [top, 2, top - 1]),
        (H.native_gate("rz", 0.7), [top]),            # stationary: no exchange
        (H.native_gate("cnot"), [top, 3]),            # control on a top qubit: no exchange
        (H.native_gate("h"), [1]),                    # shard-local
    ]


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_four_rank_group_exchange():
    import torch.multiprocessing as mp
    sys.path.insert(0, ROOT)
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    n, m, world = 8, 4, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, exchanged = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert exchanged == [1, 3, 3, 0, 3, 0, 0, 0]  # depolarising keeps both shard classes: local
    # the whole matrix, one operation at a time
    from paper_2604_15765_b200.multigpu import ShardLayout
    L = ShardLayout(n, m, 1)
    d = _tiles_to_dense(L, {0: HS.rho_payload(n, HS.rank_psi(n, 7, 4), m)}, n, m)
    for spec, tg in _ops(H, HS, n - 1):
        d = apply_kraus(d, n, spec.kraus, tg)
    want = _own_tiles(L, 0, d, m)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.linalg.norm(want)


def test_protocol_detects_missing_exchange():
    """Negative control of the emulation: without the partner's tiles, an op that moves a top qubit
    leaves NaN in the rank's own tiles (so the 4-rank test would catch a mask that is too small)."""
    sys.path.insert(0, ROOT)
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import ShardLayout
    n, m = 8, 4
    L = ShardLayout(n, m, 4)
    full = HS.rho_payload(n, HS.rank_psi(n, 7, 4), m)
    mine = L.scatter(full)[1]
    for spec, tg, needs in ((H.native_gate("cnot"), [3, 7], True), (H.native_gate("cnot"), [7, 3], False),
                            (H.native_gate("rz", 0.3), [6], False), (H.depolarising(0.2), [6], False),
                            (H.native_gate("h"), [6], True)):
        d = apply_kraus(_tiles_to_dense(L, {1: mine}, n, m), n, spec.kraus, tg)
        assert np.isnan(_own_tiles(L, 1, d, m)).any() == needs, (spec.name, tg)
