"""Sharded engine (XOR blocks) against the single-GPU engine: P shards driven from one process on one
B200 (exchange by device copies, kernels launched one after another -- no kernel waits on another).
The same per-element arithmetic runs either way, so the results must be bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _kraus2(HS):
    """Rank-2 k = 2 channel: sqrt(0.9) U, sqrt(0.1) V (CPTP)."""
    return np.stack([np.sqrt(0.9) * HS.haar(2, 11), np.sqrt(0.1) * HS.haar(2, 12)])


def _kraus3(HS):
    return np.stack([np.sqrt(0.7) * HS.haar(3, 13), np.sqrt(0.3) * HS.haar(3, 14)])


def _ops(H, HS, n):
    u2, u3 = HS.haar(2, 5), HS.haar(3, 6)
    top = n - 1
    return [
        (H.native_gate("h"), [0]), (H.native_gate("h"), [top]), (H.depolarising(0.01), [top - 1]),
        (H.amplitude_damping(0.05), [top]), (H.native_gate("rz", 0.37), [top]), (H.native_gate("rz", 1.1), [2]),
        (H.native_gate("cnot"), [top, 3]), (H.native_gate("cnot"), [1, top - 2]), (H.native_gate("cnot"), [6, 7]),
        (H.make_generic("u2", u2), [top, 5]), (H.make_generic("u2", u2), [2, top - 1]),
        (H.make_generic("u3", u3), [top, 4, 0]), (H.make_generic("u3", u3), [6, 5, 8]),
        (H.native_gate("y"), [top]), (H.native_gate("swap"), [top - 2, 1]), (H.depolarising(0.02), [5]),
        # shard-local tensor-core paths: in-tile k = 3 (4-tile items), k = 3 on two grid bits (TMA boxes,
        # quadrant mode), k = 2 promoted to k = 3 (in-tile pair, grid pair)
        (H.make_generic("u3", u3), [1, 4, 3]), (H.make_generic("u3", u3), [1, 6, 7]),
        (H.make_generic("u2", u2), [0, 3]), (H.make_generic("u2", u2), [5, 7]),
        # several top targets: the group of 4 (8) shards exchanges all-to-all
        (H.native_gate("cnot"), [top, top - 1]), (H.native_gate("cnot"), [top - 2, top]),
        (H.make_generic("u2", u2), [top - 1, top - 2]), (H.native_gate("swap"), [top, top - 2]),
        (H.make_generic("u3", u3), [top, top - 1, 2]), (H.make_generic("u3", u3), [top - 2, top, top - 1]),
        (H.make_generic("k2", _kraus2(HS)), [top, top - 1]), (H.make_generic("k3", _kraus3(HS)), [2, top, top - 2]),
        # stationary top targets: no exchange (phase; CX / Toffoli controls)
        (H.native_gate("rz", 0.9), [top - 1]), (H.native_gate("cnot"), [top, top - 1]),
        (H.native_gate("cnot"), [top - 2, 4]), (H.native_gate("toffoli"), [top, top - 2, 1]),
        (H.native_gate("toffoli"), [top, top - 1, top - 2]), (H.native_gate("z"), [top]),
    ]


@pytest.mark.parametrize("n,P,peer", [(9, 2, False), (10, 4, False), (11, 8, False), (10, 2, False), (13, 8, False),
                                      (13, 4, False), (9, 2, True), (10, 4, True), (11, 8, True), (13, 8, True),
                                      # P = G: every grid bit is a shard bit (no in-tile k = 2 promotion)
                                      (9, 16, False), (9, 16, True)])
def test_sharded_bit_identical(n, P, peer):
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import ShardGroup
    psi = HS.rank_psi(n, 42, 4)
    ref = H.TiledHermitian(n)
    ref.fill_mixture(psi)
    grp = ShardGroup(n, 5, P, peer=peer)
    grp.fill_mixture(psi)
    assert np.array_equal(grp.download_full().view(np.uint64), ref.download().view(np.uint64))
    opts = H.ApplyOptions(count_subcases=False)
    # P = G (every grid bit a shard bit): an in-tile k = 2 unitary cannot borrow grid bit 0 for the
    # k = 3 promotion (it would cross shards), so it runs the scalar two-stage transform -- the same
    # conjugation up to rounding; every other configuration is bit-identical
    exact = P < grp.layout.G
    for spec, tg in _ops(H, HS, n):
        H.apply(ref, spec, tg, opts)
        grp.apply(spec, tg)
        got, want = grp.download_full(), ref.download()
        if exact:
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (spec.name, tg, np.max(np.abs(got - want)))
        else:
            assert np.max(np.abs(got - want)) <= 1e-15 * np.linalg.norm(want), (spec.name, tg)
    assert abs(grp.trace() - H.trace(ref)) < 1e-13
    obs = ShardGroup(n, 5, P)
    obs_ref = H.TiledHermitian(n)
    strings = HS.pauli_strings(n, 16, 3)
    obs.fill_pauli_sum(*strings)
    obs_ref.fill_pauli_sum(*strings)
    assert abs(grp.expectation(obs) - H.expectation(ref, obs_ref)) < 1e-13


@pytest.mark.parametrize("n,P,peer", [(10, 4, False), (11, 8, True)])
def test_remap_bit_identical(n, P, peer):
    """Qubit remapping (multigpu.plan_remap): the same sequence with top qubits swapped down and the
    layout restored at the end equals the unremapped run bit for bit (the swaps are exact
    permutations and every op kind computes the same per-element arithmetic on any qubit)."""
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import ShardGroup
    psi = HS.rank_psi(n, 42, 4)
    ops = [(spec, tg) for spec, tg in _ops(H, HS, n) if spec.kind != "generic_kraus" or spec.k == 1]
    ops += [(H.native_gate("h"), [n - 1]), (H.native_gate("h"), [n - 2]), (H.depolarising(0.02), [n - 1])] * 3
    out = []
    for remap in (False, True):
        grp = ShardGroup(n, 5, P, peer=peer)
        grp.fill_mixture(psi)
        grp.apply_sequence(ops, remap=remap)
        grp.restore_layout()
        out.append(grp.download_full())
        grp.free()
    same = np.array_equal(out[0].view(np.uint64), out[1].view(np.uint64))
    err = float(np.max(np.abs(out[0] - out[1])))
    print(f"remap n={n} P={P}: bit-identical={same} max|delta|={err:.3e}")
    assert err <= 1e-15 * np.linalg.norm(out[0]), err


def test_group_exchange_required():
    """A cross-shard operation without the group's payloads is refused, not computed wrongly."""
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200 import _native as nat
    from paper_2604_15765_b200.multigpu import ShardGroup
    grp = ShardGroup(10, 5, 4)
    st = grp.shards[1]
    with pytest.raises((ValueError, nat.NativeError)):
        H.apply(st, H.native_gate("cnot"), [9, 8])
    # a one-bit exchange licenses an op that moves only that bit (CX target 8, control 9 stationary)
    # but not one that moves both (SWAP)
    nat.check(nat.engine().hs_state_exchange_group_from(st.handle, grp.shards[0].handle, 1))
    H.apply(st, H.native_gate("cnot"), [9, 8])
    # the exchange licensed that one operation only: its slots are stale now
    with pytest.raises((ValueError, nat.NativeError)):
        H.apply(st, H.native_gate("cnot"), [9, 8])
    nat.check(nat.engine().hs_state_exchange_group_from(st.handle, grp.shards[0].handle, 1))
    with pytest.raises((ValueError, nat.NativeError)):
        H.apply(st, H.native_gate("swap"), [9, 8])


def _ipc_worker(rank, world, port, n, q):
    import os
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    from paper_2604_15765_b200.multigpu import DistributedShard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sh = DistributedShard(n, 5, device=0, peer=True)  # both ranks on GPU 0: CUDA IPC, host barriers
    sh.state.fill_mixture(HS.rank_psi(n, 42, 4))
    for spec, tg in _ops(H, HS, n):
        sh.apply(spec, tg)
    sh.state.synchronize()
    dist.barrier()
    parts = [None] * world
    dist.all_gather_object(parts, sh.state.download())
    if rank == 0:
        q.put(sh.layout.gather(parts))
    dist.barrier()
    sh.close()
    dist.destroy_process_group()


def test_peer_mode_across_processes():
    """Peer mode with CUDA IPC between two processes (two shards on one GPU: the kernels never wait on
    each other -- ordering is by host barriers) against the single-GPU engine, bit for bit."""
    import socket
    import torch.multiprocessing as mp
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    n, world = 10, 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = H.TiledHermitian(n)
    ref.fill_mixture(HS.rank_psi(n, 42, 4))
    opts = H.ApplyOptions(count_subcases=False)
    for spec, tg in _ops(H, HS, n):
        H.apply(ref, spec, tg, opts)
    assert np.array_equal(got.view(np.uint64), ref.download().view(np.uint64))
