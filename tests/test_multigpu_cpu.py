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


def _seq(H, HS, n):
    """Every op kind of the sharded engine tests (tests/test_multigpu_gpu.py::_ops), at n qubits."""
    u2, u3 = HS.haar(2, 5), HS.haar(3, 6)
    top = n - 1
    k2 = np.stack([np.sqrt(0.9) * HS.haar(2, 11), np.sqrt(0.1) * HS.haar(2, 12)])
    return [
        (H.native_gate("h"), [0]), (H.native_gate("h"), [top]), (H.depolarising(0.01), [top - 1]),
        (H.amplitude_damping(0.05), [top]), (H.native_gate("rz", 0.37), [top]), (H.native_gate("cnot"), [top, 3]),
        (H.native_gate("cnot"), [1, top - 1]), (H.make_generic("u2", u2), [top, 2]),
        (H.make_generic("u3", u3), [top, 4, 0]), (H.native_gate("y"), [top]), (H.native_gate("swap"), [top - 1, 1]),
        (H.native_gate("cnot"), [top, top - 1]), (H.make_generic("u2", u2), [top - 1, top]),
        (H.make_generic("k2", k2), [top, top - 1]), (H.native_gate("toffoli"), [top, top - 1, 2]),
        (H.native_gate("h"), [top - 1]), (H.native_gate("h"), [top]), (H.native_gate("h"), [top - 1]),
    ]


def _worker(rank, world, port, n, peer, remap, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import shard_emu
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import DistributedShard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    be = shard_emu.EmuBackend()
    sh = DistributedShard(n, 5, device=0, peer=peer, remap=remap, backend=be)
    full = HS.rho_payload(n, HS.rank_psi(n, 17, 4))
    sh.state.upload(sh.layout.scatter(full)[rank])
    sh.apply_sequence(_seq(H, HS, n))
    if remap:
        sh.restore_layout()
    tr = sh.reduce(None, 2)
    parts = [None] * world
    dist.all_gather_object(parts, sh.state.download())
    ex = [None] * world
    dist.all_gather_object(ex, sh.exchanges)
    if rank == 0:
        q.put((sh.layout.gather(parts), tr, ex))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, n, peer, remap):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, peer, remap, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("world,n,peer", [(2, 7, False), (4, 8, False), (4, 8, True)])
def test_distributed_shard_gloo(world, n, peer):
    """multigpu.DistributedShard itself on `world` CPU ranks over gloo (device side emulated by
    tests/shard_emu.py): each rank holds only its shard, exchanges what op_mask names, and the
    gathered operator equals the dense evolution of the whole matrix."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import shard_emu
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    got, tr, ex = _run(world, n, peer, remap=False)
    from paper_2604_15765_b200.multigpu import ShardLayout
    L = ShardLayout(n, 5, world)
    full = HS.rho_payload(n, HS.rank_psi(n, 17, 4))
    dense = shard_emu.tiles_to_dense(L, dict(enumerate(L.scatter(full))), n, 5)
    for spec, tg in _seq(H, HS, n):
        dense = shard_emu.apply_kraus_dense(dense, n, spec.kraus, tg)
    want = L.gather([shard_emu.own_tiles(L, s, dense, 5) for s in range(world)])
    assert np.max(np.abs(got - want)) <= 1e-13 * np.linalg.norm(dense)
    assert abs(tr - np.trace(dense).real) < 1e-12
    assert min(ex) > 0  # cross-shard ops did exchange


def test_distributed_shard_remap_gloo():
    """Qubit remapping (multigpu.plan_remap) on 4 gloo ranks: swaps inserted, the layout restored at
    the end, the same operator as the unremapped run.  (The emulator's dense block sums run in an
    axis order that follows the physical qubits, so agreement is to rounding here; the engine's
    bit-identity under remapping is tests/test_multigpu_gpu.py::test_remap_bit_identical.)"""
    got0, tr0, ex0 = _run(4, 8, False, remap=False)
    got1, tr1, ex1 = _run(4, 8, False, remap=True)
    assert np.max(np.abs(got0 - got1)) <= 1e-15 * np.linalg.norm(got0) * 2
    print("exchanges per rank: plain", ex0, "remapped (incl. swaps and restore)", ex1)


def test_plan_remap_counts():
    """plan_remap on C4's sequence (n = 17, 8 shards): logical results unchanged (the actions are a
    valid relabelling) and the exchange count with remapping never exceeds the plain one."""
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import ShardLayout, plan_remap
    n = 17
    L = ShardLayout(n, 5, 8)
    ops = []
    for op in HS.config_ops("c4", n)[:118]:
        spec = {"h": lambda: H.native_gate("h"), "cnot": lambda: H.native_gate("cnot"),
                "rz": lambda: H.native_gate("rz", op.param), "depol": lambda: H.depolarising(op.param)}[op.kind]()
        ops.append((spec, list(op.targets)))
    perm = list(range(n))
    actions, plain, remapped = plan_remap(ops, L, perm)
    assert sum(1 for a in actions if a[0] == "op") == len(ops)
    assert remapped <= plain
    assert sorted(perm) == list(range(n))


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
