"""Host logic of the multi-GPU path on CPU: the shard layout (bijective, balanced, the reference layout
at P = 1), the exchange plan, and a 2-rank gloo run in which every rank holds only its shard,
exchanges with its partner over torch.distributed for the cross-shard qubit, applies the per-shard
unit rule (tests/shard_emu.py), and the gathered result matches the oracle."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _layout(n, m, P):
    from paper_2604_15765_b200.multigpu import ShardLayout
    return ShardLayout(n, m, P)


@pytest.mark.parametrize("n,m,P", [(8, 5, 1), (9, 5, 2), (10, 5, 4), (11, 5, 8), (9, 2, 8), (12, 5, 8)])
def test_layout_bijective_and_balanced(n, m, P):
    L = _layout(n, m, P)
    G = L.G
    seen = {}
    for s in range(P):
        for t in range(L.tiles(s)):
            ti, tj = L.decode(s, t)
            assert ti >= tj and L.shard_of(ti, tj) == s and L.index(ti, tj, s) == t
            seen[(ti, tj)] = s
    assert len(seen) == G * (G + 1) // 2
    sizes = [L.tiles(s) for s in range(P)]
    assert max(sizes) / (sum(sizes) / P) <= 1 + 1 / L.B + 1e-12
    if P == 1:
        assert all(L.index(ti, tj) == ti * (ti + 1) // 2 + tj for ti in range(G) for tj in range(ti + 1))


def test_partner_plan():
    L = _layout(11, 5, 8)  # G = 64, top qubits 8, 9, 10
    assert L.top0 == 8
    assert L.partner(3, [0]) == -1 and L.partner(3, [7, 2]) == -1
    assert L.partner(3, [8]) == 2 and L.partner(3, [9]) == 1 and L.partner(3, [10, 1]) == 7
    with pytest.raises(ValueError):
        L.partner(0, [8, 9])
    # two or three top targets couple the group s ^ span(mask)
    assert L.group_mask([9, 8]) == 3 and L.group_mask([10, 3, 8]) == 5 and L.group_mask([1, 2]) == 0
    assert L.group(3, [9, 8]) == [3, 2, 1, 0] and L.group(6, [10, 2, 8]) == [6, 7, 2, 3]
    assert L.group(5, [10, 9, 8]) == [5 ^ d for d in range(8)]
    # a k = 2 unit on two top qubits spans exactly its group of four shards
    for ti in range(0, 64, 5):
        for tj in range(ti + 1):
            if (ti | tj) >> 3 & 3:
                continue
            sh = {L.shard_of(max(a, b), min(a, b)) for a in (ti, ti | 8, ti | 16, ti | 24)
                  for b in (tj, tj | 8, tj | 16, tj | 24)}
            s0 = min(sh)
            assert sh == {s0 ^ d for d in range(4)}
    # a k = 1 cross unit spans exactly the pair (s, s ^ 2^c) (SURVEY 8e XOR-block property)
    for c, q in ((0, 8), (1, 9), (2, 10)):
        ap = q - 5
        for ti in range(64):
            for tj in range(ti + 1):
                if (ti >> ap) & 1 or (tj >> ap) & 1:
                    continue
                sh = {L.shard_of(max(a, b), min(a, b)) for a in (ti, ti | 1 << ap) for b in (tj, tj | 1 << ap)}
                assert len(sh) == 2 and (min(sh) ^ max(sh)) == 1 << c


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, n, ops, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import shard_emu
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200.multigpu import ShardLayout
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    L = ShardLayout(n, 5, world)
    full = HS.rho_payload(n, HS.rank_psi(n, 17, 4))
    mine = L.scatter(full)[rank].copy()
    for name, srow, a in ops:
        partner = L.partner(rank, [a])
        recv = None
        if partner >= 0:
            buf = torch.from_numpy(np.zeros(L.count(partner), np.complex128).view(np.float64))
            send = torch.from_numpy(mine.view(np.float64).copy())
            for r in (dist.isend(send, partner), dist.irecv(buf, partner)):
                r.wait()
            recv = buf.numpy().view(np.complex128)
        shard_emu.apply_k1(L, rank, mine, recv, srow, a)
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        q.put(L.gather(parts))
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_channels(oracle, orc):
    import torch.multiprocessing as mp
    from paper_2604_15765_b200 import harness as HS
    n, world = 8, 2
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    chans = [("depol", oracle.depolarising(0.1)), ("ampdamp", oracle.amplitude_damping(0.2)), ("h", oracle.generic(h))]
    seq = [(0, 7), (1, 7), (2, 3), (0, 6), (1, 5), (2, 7)]  # (channel, qubit); 7 is the cross-shard qubit
    ops = []
    for ci, a in seq:
        s = orc.transfer_from_kraus(chans[ci][1].ops)
        srow = np.zeros((4, 4), np.complex128)
        for i in range(2):
            for ip in range(2):
                for mu in range(2):
                    for nu in range(2):
                        srow[i * 2 + ip, mu * 2 + nu] = s[i + ip * 2, mu + nu * 2]  # kernels.cpp:27-37
        ops.append((chans[ci][0], srow, a))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, ops, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = HS.rho_payload(n, HS.rank_psi(n, 17, 4))
    for ci, a in seq:
        orc.apply(want, n, 5, chans[ci][1], [a])
    assert oracle.rel_max_err(got, want, orc.frobenius(want, n, 5)) <= 1e-13


def test_exchange_mask_moving_bits():
    """Only qubits an op moves need the partner's tiles: a phase never, a CX only its target."""
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import ShardLayout, moving_qubits, op_mask
    L = ShardLayout(11, 5, 8)  # top qubits 8, 9, 10 -> shard bits 0, 1, 2
    cx, rz, h, sw = H.native_gate("cnot"), H.native_gate("rz", 0.4), H.native_gate("h"), H.native_gate("swap")
    assert moving_qubits(rz, [10]) == set() and op_mask(L, rz, [10]) == 0
    assert moving_qubits(cx, [10, 3]) == {3} and op_mask(L, cx, [10, 3]) == 0      # control on a top qubit
    assert moving_qubits(cx, [3, 10]) == {10} and op_mask(L, cx, [3, 10]) == 4     # target on a top qubit
    assert op_mask(L, cx, [10, 9]) == 2 and op_mask(L, sw, [10, 9]) == 6
    assert op_mask(L, h, [9]) == 2 and op_mask(L, H.native_gate("toffoli"), [10, 9, 8]) == 1
    assert op_mask(L, H.depolarising(0.1), [8]) == 0  # (00,11)/(01,10) couplings only: shard-local
    assert op_mask(L, H.amplitude_damping(0.2), [9]) == 0
    k = np.stack([np.eye(2) * np.sqrt(0.9), np.sqrt(0.1) * np.array([[1, 1], [1, -1]]) / np.sqrt(2)])
    assert op_mask(L, H.make_generic("mix_h", k), [9]) == 2  # couples the classes: exchange
