#!/usr/bin/env python3
"""Benchmark of the hot path (BASELINE.json metric: gate conjugations/s and achieved HBM GB/s as a
fraction of the roofline, n = 16, fp64).

Default workload = config C2 (BASELINE.json configs[2], the n = 16 single-GPU config the metric is
quoted on): depolarising(p = 0.01) then amplitude damping(gamma = 0.05) on every qubit of an n = 16
complex128 density matrix (rank-4, seeded) in the tiled lower-triangle layout, m = 5 (34.38 GB
stored).  A step = one pass of the 32 channel applications.

  python bench.py [--gpus N --steps K --warmup W] [--config c0..c4] [--impl ours|reference]

* value      ops/s over all ranks, state resident in HBM, CUDA events on the engine's stream, max
             over ranks.  The 34 GB state is far larger than the 126 MB L2, so no flush is needed.
* e2e        the same metric through the public API with the state in pinned HOST memory: each
             step uploads the payload, applies the 32 ops and downloads the result.
* roofline   achieved = algorithmic bytes per launch (2 x stored bytes: one read + one write of the
             triangle) / mean launch duration (events around every launch); peak from
             MEASURED_PEAKS.json; traffic = ncu dram bytes per launch from profiles/ (if captured).
* cpu_baseline  the reference library itself (oracle/_ref/libhermsim_ref.so, built from
             /root/reference) timed on this host on a bounded sample of the same workload.
* --impl reference  times that reference CPU path alone, all host threads (rank 0 only).
For N > 1 (torchrun) the operator is partitioned into N XOR-block shards, one per GPU (strong
scaling; value = ops of the one operator per second); a cross-shard op's kernels read the group
members' tiles in place over NVLink (peer mode, CUDA IPC) or, with --exchange, after an NCCL group
exchange.  --remap adds qubit remapping (multigpu.plan_remap); --replicas runs N independent copies
instead (weak scaling).  roofline_nvlink: remote bytes a cross-shard op reads / its time / the
measured NVLink peer bandwidth (B200_PROFILING.md: 770 GB/s per direction).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gate conjugations/sec and achieved HBM GB/s (fraction of roofline), n=16 fp64"
UNIT = "gate conjugations/s"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
NVLINK_GBS = 770.0  # B200_PROFILING.md: measured peer copy, per direction per GPU (900 nominal)
# FP64 tensor (DMMA) peak: measured on B200 by tools/fp64_probe.cu (profiles/r01_fp64_probe.txt:
# m8n8k4, 8-32 warps/SM, 37.0-37.1 TFLOP/s; DFMA shares the pipe at 36.8)
FP64_TFLOPS = 37.1


def fp64_fma_per_element(op) -> int:
    """Algorithmic FP64 FMAs per stored element of one op's transform (DESIGN.md 4.2 / 4.5): the
    k = 3 direct form L B L^dagger in 3M form 48; a k = 2 unitary through I2 (x) L on the k = 3
    path 48; the k = 2 Kraus S form (16 x 16, 3M) 48; a k = 3 Kraus sum of rank 2 as two direct
    conjugations 96; rank >= 3 in the hermitian basis (two real 64 x 64 products per block) 128;
    single-qubit ops and permutations are HBM streams (<= 16, counted 0)."""
    k = len(op.targets)
    if op.kind in ("unitary", "unitary_dual"):
        return 48 if k >= 2 else 0
    if op.kind == "kraus":
        r = op.matrix.shape[0]
        if k == 3:
            return 48 if r == 1 else 96 if r == 2 else 128
        if k == 2:
            return 48
    return 0

WORKLOADS = {
    "c0": "C0: Hadamard at qubits 0..11 (12 ops) on an n=12 rank-4 rho, m=5",
    "c1": "C1: CX then Haar U4 on all 182 ordered pairs (364 ops) on an n=14 rank-4 rho, m=5",
    "c2": "C2: depolarising(0.01) then amplitude damping(0.05) on qubits 0..15 (32 ops) on an n=16 rank-4 rho, m=5",
    "c3": "C3: 20 layers x 5 Haar 8x8 blocks in the Heisenberg picture (100 ops) on an n=16 Pauli-sum O, m=5",
    "c4": "C4: 10 layers of Rz+H per qubit, CX matching, depolarising(0.001) (590 ops) on an n=17 rank-4 rho, m=5",
    "kraus": ("KRAUS: 2 layers of [two-qubit depolarising(0.01) (rank 16) on 8 seeded pairs, seeded random rank-4 "
              "three-qubit channels on 5 seeded triples] (26 Kraus-sum passes) on an n=16 rank-4 rho, m=5"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- distributed
def dist_setup():
    """One rank per GPU over NCCL.  BENCH_FUNCTIONAL_ONE_GPU=1 (code-path check only, never a
    measurement): every rank on GPU 0 with a gloo group -- the sharded peer mode then orders the
    ranks by host barriers, so no kernel waits on another."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("BENCH_FUNCTIONAL_ONE_GPU") == "1":
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def dist_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if dist.get_backend() == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_min(x: float, world: int) -> float:
    return -dist_max(-x, world)


def dist_barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------------------ workloads
def build_ops(H, HS, cfg: str, n: int):
    """Op list -> [(spec, targets, label)] through the public API (ChannelSpec objects)."""
    specs = {}
    out = []
    for op in HS.config_ops(cfg, n):
        if op.kind == "h":
            spec = specs.setdefault("h", H.native_gate("h"))
        elif op.kind == "cnot":
            spec = specs.setdefault("cnot", H.native_gate("cnot"))
        elif op.kind == "rz":
            spec = H.native_gate("rz", op.param)
        elif op.kind == "depol":
            spec = specs.setdefault(("depol", op.param), H.depolarising(op.param))
        elif op.kind == "ampdamp":
            spec = specs.setdefault(("amp", op.param), H.amplitude_damping(op.param))
        elif op.kind == "unitary":
            spec = H.make_generic("haar", op.matrix)
        elif op.kind == "unitary_dual":
            spec = H.dual_channel(H.make_generic("haar", op.matrix))
        elif op.kind == "kraus":
            spec = H.make_generic("kraus", op.matrix)
        else:
            raise ValueError(op.kind)
        out.append((spec, list(op.targets), op.kind))
    return out


def host_payload(HS, n, m, psi, out: np.ndarray | None = None, threads: int | None = None) -> np.ndarray:
    """Tiled payload of the rank-4 rho built on the host by the harness, multi-threaded."""
    cnt = HS.payload_count(n, m)
    if out is None:
        out = np.empty(cnt, np.complex128)
    G = (1 << n) >> m if n >= m else 1
    T = G * (G + 1) // 2
    threads = threads or os.cpu_count() or 1
    bounds = [T * i // threads for i in range(threads + 1)]
    from paper_2604_15765_b200 import _native as nat
    L = nat.harness()
    psi = np.ascontiguousarray(psi)

    def work(i):
        t0, t1 = bounds[i], bounds[i + 1]
        if t1 > t0:
            view = out[t0 << (2 * m): t1 << (2 * m)]
            L.hsg_rho_payload_range(n, m, psi.shape[0], psi.ctypes.data_as(nat.c_double_p),
                                    view.ctypes.data_as(nat.c_double_p), t0, t1)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return FALLBACK_HBM_GBS, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"


def traffic_key(cfg: str, n: int, shards: int = 1) -> str:
    return f"{cfg}:n{n}" + (f":p{shards}" if shards > 1 else "")


def load_traffic(cfg: str, n: int, shards: int = 1):
    """ncu DRAM bytes per launch of the config's dominant kernel, captured at exactly this (config,
    n, shards) (profiles/ncu_traffic.json); None when no capture matches."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    e = d.get(traffic_key(cfg, n, shards))
    if not e:
        return None, None
    return e.get("traffic_bytes_per_launch"), e.get("source")


# --------------------------------------------------------------------------- reference arm
def stratified_order(nblocks: int) -> list[int]:
    """Block indices in van der Corput order (bit-reversed counter): every prefix of the order is
    spread evenly over the sequence, so a short timed sample covers all qubit positions alike."""
    bits = max(1, (nblocks - 1).bit_length())
    out = []
    for i in range(1 << bits):
        b = int(format(i, f"0{bits}b")[::-1], 2)
        if b < nblocks:
            out.append(b)
    return out


def ref_channel(O, op):
    if op.kind == "h":
        return O.native_gate("h")
    if op.kind == "cnot":
        return O.native_gate("cnot")
    if op.kind == "rz":
        return O.native_gate("rz", op.param)
    if op.kind == "depol":
        return O.depolarising(op.param)
    if op.kind == "ampdamp":
        return O.amplitude_damping(op.param)
    if op.kind == "unitary":
        return O.generic(op.matrix)
    if op.kind == "unitary_dual":
        return O.dual(O.generic(op.matrix))
    if op.kind == "kraus":
        return O.generic(op.matrix)
    raise ValueError(op.kind)


def run_reference_cpu(cfg: str, n: int, m: int, fill, ops_per_step: int, steps: int, warmup: int, threads: int,
                      budget_s: float | None = None):
    """Times the compiled reference (hermsim::apply, threads = host cores).  The state is built in
    the reference's own buffer by `fill(view)` (no second host copy: n = 17 is 137.5 GB).  A step is
    a block of `ops_per_step` consecutive ops of the config's sequence; the timed steps take the
    blocks in stratified order (stratified_order) from the start, the warm-up steps take blocks from
    the end of that order, so warm-up never displaces a position from the timed sample.
    Returns (times, blocks, ops_total)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2604_15765_b200 import harness as HS
    ref = O.Reference()
    h = ref.create(n, m)
    fill(ref.view(h))
    seq = HS.config_ops(cfg, n)
    nblocks = max(1, len(seq) // ops_per_step)
    order = stratified_order(nblocks)
    chans = {}
    times, used = [], []
    t_start = time.perf_counter()
    plan = [order[-1 - (w % len(order))] for w in range(warmup)] + [order[k % len(order)] for k in range(steps)]
    for s, b in enumerate(plan):
        t0 = time.perf_counter()
        for op in seq[b * ops_per_step:(b + 1) * ops_per_step]:
            key = (op.kind, op.param, id(op.matrix) if op.matrix is not None else None)
            ch = chans.get(key)
            if ch is None:
                ch = chans[key] = ref_channel(O, op)
            ref.apply(h, ch, list(op.targets), threads=threads)
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
            used.append(b)
        if budget_s is not None and time.perf_counter() - t_start > budget_s and len(times) >= 1:
            break
    ref.free(h)
    targets = sorted({q for b in used for op in seq[b * ops_per_step:(b + 1) * ops_per_step] for q in op.targets})
    return times, used, targets


def reference_fill(HS, cfg, n, m, threads, psi=None, strings=None):
    """Callback building the config's seeded input in place (the reference's buffer)."""
    seed = HS.SEEDS[cfg]

    def fill(view):
        if cfg == "c3":
            view[:] = HS.pauli_payload(n, strings if strings is not None else HS.pauli_strings(n, 64, seed), 5)
        else:
            host_payload(HS, n, m, psi if psi is not None else HS.rank_psi(n, seed, 4), out=view, threads=threads)
    return fill


# --------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--qubits", "--n", dest="n", type=int, default=None, help="override the config's qubit count (testing)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--e2e-states", type=int, default=4,
                    help="device states / pinned host buffers in flight in the pipelined e2e loop (as memory allows)")
    ap.add_argument("--e2e-serial", action="store_true",
                    help="e2e without overlapping consecutive steps (one state, one buffer)")
    ap.add_argument("--shard", dest="shard", action="store_true", default=None,
                    help="partition the operator over the N ranks (the default when N > 1)")
    ap.add_argument("--replicas", dest="shard", action="store_false", help="N independent replicas (weak scaling)")
    ap.add_argument("--remap", action="store_true",
                    help="sharded: qubit remapping (swap top qubits that keep needing exchanges with low ones)")
    ap.add_argument("--remap-window", type=int, default=64, help="remapping lookahead (operations)")
    ap.add_argument("--exchange", action="store_true",
                    help="sharded: NCCL exchange of the group's shards before a cross-shard op (default: peer mode, "
                         "the op's kernels read the members' tiles in place over NVLink)")
    ap.add_argument("--graph", action="store_true",
                    help="capture one step as a CUDA graph after the warm-up and replay it (hermsim.capture)")
    ap.add_argument("--fuse", action="store_true",
                    help="operation fusion (SURVEY 8f): same sequence, fewer passes; value counts the logical ops")
    args = ap.parse_args()

    from paper_2604_15765_b200 import harness as HS

    cfg = args.config
    n = args.n or HS.CONFIG_N[cfg]
    m = 5
    world, rank, local = (1, 0, 0)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return 0
        return reference_arm(args, cfg, n, m, world)
    world, rank, local = dist_setup()
    return ours_arm(args, cfg, n, m, world, rank, local)


def reference_arm(args, cfg, n, m, world):
    from paper_2604_15765_b200 import harness as HS
    threads = os.cpu_count() or 1
    nc = cpu_sample_n(cfg, n, m)
    ops_per_step = 2
    times, blocks, covered = run_reference_cpu(cfg, nc, m, reference_fill(HS, cfg, nc, m, threads), ops_per_step,
                                               args.steps, args.warmup, threads)
    t = float(np.mean(times))
    value = ops_per_step / t / 4.0 ** (n - nc)
    sample = (f"{ops_per_step} consecutive ops of {cfg} per step at n={nc} through hermsim::apply "
              "(oracle/_ref/libhermsim_ref.so, threads=nproc); timed blocks in stratified order over the sequence "
              f"(blocks {blocks}), warm-up blocks separate")
    if nc != n:
        sample += f"; host RAM/time-bounded, extrapolated to n={n} by 4^(n-{nc})"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": {"workload": WORKLOADS[cfg], "n": n, "m": m, "ops_per_step": ops_per_step,
                   "qubits_covered": covered},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def ours_arm(args, cfg, n, m, world, rank, local):
    from paper_2604_15765_b200 import harness as HS
    from paper_2604_15765_b200 import hermsim as H
    import ctypes
    nat = H.nat
    L = nat.engine()

    seed = HS.SEEDS[cfg]
    sharded = world > 1 and args.shard is not False
    if args.remap and not sharded:
        raise SystemExit("--remap applies to sharded runs (N > 1)")
    dshard = None
    if sharded:
        from paper_2604_15765_b200.multigpu import DistributedShard, plan_remap
        dshard = DistributedShard(n, m, device=local, peer=not args.exchange, remap=args.remap)
        st = dshard.state
        apply_op = dshard.apply
    else:
        st = H.TiledHermitian(n, m, device=local)
        apply_op = lambda spec, tg, o: H.apply(st, spec, tg, o)  # noqa: E731
    S = st.element_count() * 16  # this rank's stored bytes
    psi = None
    strings = None
    if cfg == "c3":
        strings = HS.pauli_strings(n, 64, seed)
        st.fill_pauli_sum(*strings)
        drho = DistributedShard(n, m, device=local, peer=not args.exchange) if sharded else None
        rho = drho.state if sharded else H.TiledHermitian(n, m, device=local)
        psi = HS.rank_psi(n, seed + 1, 4)
        rho.fill_mixture(psi)
    else:
        psi = HS.rank_psi(n, seed, 4)
        st.fill_mixture(psi)
    ops = build_ops(H, HS, cfg, n)
    nops = len(ops)
    opts = H.ApplyOptions(count_subcases=False)
    fplan = None
    if args.fuse:
        if sharded:
            raise SystemExit("--fuse runs on single-GPU / replica states")
        from paper_2604_15765_b200 import fusion
        fplan = fusion.plan_sequence([(spec, tg) for spec, tg, _ in ops], n, m)

    def actions_of_step():
        """The launches of one step: the ops themselves, or (remapping) ops on physical qubits with
        the planner's SWAPs in between (the map carries over from step to step)."""
        if not args.remap:
            return [("op", spec, tg) for spec, tg, _ in ops]
        acts, _, _ = plan_remap([(spec, tg) for spec, tg, _ in ops], dshard.layout, dshard.perm, args.remap_window)
        return acts

    if fplan is not None:
        npass = fplan.launches
    elif args.remap:
        npass = 4 * nops  # event slots: ops plus the planner's swaps (at most k per op)
    else:
        npass = nops
    ev = [ctypes.c_void_p() for _ in range(2 * npass + 2)]
    for e in ev:
        nat.check(L.hs_event_create(ctypes.byref(e)))

    touched = []  # per launch: HBM bytes read + written (engine plan, algorithmic), remote bytes
    remote = []

    def physical(spec, tg, o):
        if dshard is not None and args.remap:
            return dshard._apply_physical(spec, tg, o)
        return apply_op(spec, tg, o)

    def step(record=False, collect=False):
        if fplan is not None:  # fused passes; touched bytes: 2 S per pass (program or composed step)
            for i, item in enumerate(fplan.items):
                if record:
                    L.hs_event_record(ev[2 + 2 * i], st.handle)
                fusion.execute(st, fusion.Plan([item]), opts)
                if collect:
                    touched.append(2 * S)
                    remote.append(0)
                if record:
                    L.hs_event_record(ev[3 + 2 * i], st.handle)
            return len(fplan.items)
        acts = actions_of_step()
        for i, a in enumerate(acts):
            spec, tg = (a[1], a[2]) if a[0] == "op" else (None, [a[1], a[2]])
            if spec is None:
                from paper_2604_15765_b200.multigpu import _swap_spec
                spec = _swap_spec()
            if record:
                L.hs_event_record(ev[2 + 2 * i], st.handle)
            plan = physical(spec, tg, opts)
            if collect:
                tb = int(plan.touched_bytes)
                # a cross-shard op also reads its group members' tiles (the plan counts them)
                touched.append(min(tb, 2 * S))
                remote.append(max(0, tb - 2 * S))
            if record:
                L.hs_event_record(ev[3 + 2 * i], st.handle)
        return len(acts)

    for w in range(args.warmup):
        if w == 0:
            touched.clear()
            remote.clear()
        step(collect=(w == 0))
    st.synchronize()
    graph = None
    if args.graph:
        if sharded:
            raise SystemExit("--graph runs on single-GPU / replica states")
        with H.capture(st) as graph:  # per-launch events are not captured: launches share the step time
            step()
        plain_step = step

        def step(record=False, collect=False):  # noqa: F811
            graph.launch()
            return npass
        _ = plain_step
    dist_barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = H.launch_count()
    launch_ms = []
    L.hs_event_record(ev[0], st.handle)
    t_host0 = time.perf_counter()
    nlast = npass
    for s in range(args.steps):
        if s == args.steps - 1 and args.remap:  # the last step's launches are timed one by one
            touched.clear()
            remote.clear()
            nlast = step(record=True, collect=True)
        else:
            nlast = step(record=(s == args.steps - 1)) or npass
    L.hs_event_record(ev[1], st.handle)
    st.synchronize()
    t_host = time.perf_counter() - t_host0
    launches = H.launch_count() - launches0
    ms = ctypes.c_float()
    nat.check(L.hs_event_elapsed_ms(ev[0], ev[1], ctypes.byref(ms)))
    total_ms = float(ms.value)
    for i in range(nlast):
        if graph is not None:
            launch_ms.append(total_ms / args.steps / npass)
            continue
        x = ctypes.c_float()
        nat.check(L.hs_event_elapsed_ms(ev[2 + 2 * i], ev[3 + 2 * i], ctypes.byref(x)))
        launch_ms.append(float(x.value))
    clk = clocks.stop()
    dist_barrier(world)
    total_ms = dist_max(total_ms, world)
    ms_per_step = total_ms / args.steps
    value = (1 if sharded else world) * nops * args.steps / (total_ms / 1e3)

    # HBM roofline of the launches of one step (this rank): algorithmic bytes / launch durations
    peak, peak_src = load_peaks()
    if not touched:
        touched = [2 * S] * len(launch_ms)
        remote = [0] * len(launch_ms)
    touched, remote = touched[:len(launch_ms)], remote[:len(launch_ms)]
    per_launch_bytes = float(np.mean(touched))
    mean_launch_ms = float(np.mean(launch_ms))
    achieved = sum(touched) / (sum(launch_ms) / 1e3) / 1e9
    traffic, traffic_src = load_traffic(cfg, n, world if sharded else 1)
    # NVLink roofline of the cross-shard launches: remote bytes read / their durations
    xs = [(r, t) for r, t in zip(remote, launch_ms) if r > 0]
    roof_nv = None
    if sharded:
        if xs:
            nv = sum(r for r, _ in xs) / (sum(t for _, t in xs) / 1e3) / 1e9
            roof_nv = {"bound": "nvlink", "achieved": nv, "peak": NVLINK_GBS, "unit": "GB/s", "frac": nv / NVLINK_GBS,
                       "cross_shard_launches_per_step": len(xs),
                       "remote_bytes_per_cross_launch": float(np.mean([r for r, _ in xs])),
                       "mean_cross_launch_ms": float(np.mean([t for _, t in xs])),
                       "peak_source": "B200_PROFILING.md: measured peer copy 770 GB/s per direction (900 nominal)",
                       "mode": "NCCL group exchange + op" if args.exchange else "peer reads fused into the op kernels"}
        else:
            roof_nv = {"bound": "nvlink", "achieved": None, "frac": None, "cross_shard_launches_per_step": 0,
                       "note": "no operation of this config reads another shard's tiles (single-qubit channels "
                               "that keep the (00,11)/(01,10) shard classes apart run shard-local)"}
    # min(HBM, FP64) roofline for configs with FP64-heavy transforms (k = 3 Kraus sums): each launch
    # is bound by max(bytes / HBM peak, flops / DMMA peak); frac = sum of bounds / sum of launch times
    roof_mixed = None
    seq = HS.config_ops(cfg, n)
    if fplan is None and not args.remap and len(seq) == len(launch_ms):
        elems = S / 16.0
        fl = [2.0 * fp64_fma_per_element(op) * elems for op in seq]
        if any(fl):
            bounds = [max(tb / (peak * 1e9), f / (FP64_TFLOPS * 1e12)) for tb, f in zip(touched, fl)]
            nfp = sum(1 for tb, f in zip(touched, fl) if f / (FP64_TFLOPS * 1e12) > tb / (peak * 1e9))
            fp_t = sum(t for t, tb, f in zip(launch_ms, touched, fl) if f / (FP64_TFLOPS * 1e12) > tb / (peak * 1e9))
            fp_f = sum(f for tb, f in zip(touched, fl) if f / (FP64_TFLOPS * 1e12) > tb / (peak * 1e9))
            roof_mixed = {"bound": "max(hbm, fp64) per launch", "frac": sum(bounds) / (sum(launch_ms) / 1e3),
                          "hbm_peak_gbs": peak, "fp64_peak_tflops": FP64_TFLOPS,
                          "fp64_bound_launches_per_step": nfp,
                          "fp64_achieved_tflops": (fp_f / (fp_t / 1e3) / 1e12) if fp_t else None,
                          "fp64_peak_source": "tools/fp64_probe.cu on B200 (profiles/r01_fp64_probe.txt), DMMA m8n8k4",
                          "flops_model": "bench.fp64_fma_per_element x 2 x stored elements"}
    result = {}
    if cfg == "c3":
        result["tr_rho_O"] = drho.reduce(dshard, 0) if sharded else H.expectation(rho, st)

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    hbuf = ctypes.c_void_p()
    if not args.no_e2e:
        got = L.hs_host_alloc(ctypes.c_uint64(S), ctypes.byref(hbuf)) == 0
        if dist_min(1.0 if got else 0.0, world) < 1.0:  # every rank measures, or none does
            log("e2e skipped: a pinned host buffer of %.1f GB is not available on every rank" % (S / 1e9))
            if got:
                L.hs_host_free(hbuf)
            hbuf = None
    if not args.no_e2e and hbuf is not None:
        host = np.ctypeslib.as_array(ctypes.cast(hbuf, ctypes.POINTER(ctypes.c_double)), shape=(2 * st.element_count(),))
        nat.check(L.hs_state_download(st.handle, host.ctypes.data_as(nat.c_double_p), st.element_count()))
        e2e = None
        # overlapped steps (extra device states and pinned buffers) on a single-GPU run; with N ranks
        # on one node each rank keeps one pinned payload-sized buffer
        if not sharded and not args.e2e_serial and world == 1:
            e2e = pipelined_e2e(args, H, L, nat, st, host, S, n, m, nops, world, fplan, ops, opts)
        if e2e is None:
            e_ms = []
            for s in range(1 + args.e2e_steps):
                dist_barrier(world)
                L.hs_event_record(ev[0], st.handle)
                nat.check(L.hs_state_upload_async(st.handle, host.ctypes.data_as(nat.c_double_p), st.element_count()))
                step()
                nat.check(L.hs_state_download_async(st.handle, host.ctypes.data_as(nat.c_double_p), st.element_count()))
                L.hs_event_record(ev[1], st.handle)
                st.synchronize()
                x = ctypes.c_float()
                nat.check(L.hs_event_elapsed_ms(ev[0], ev[1], ctypes.byref(x)))
                if s >= 1:
                    e_ms.append(float(x.value))
            e2e_ms = dist_max(float(np.mean(e_ms)), world)
            job_bytes = S * (world if sharded else 1)
            e2e = {"value": (1 if sharded else world) * nops / (e2e_ms / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": job_bytes, "d2h_bytes_per_step": job_bytes,
                   "h2d_bytes_per_step_per_rank": S, "ms_per_step": e2e_ms, "steps": len(e_ms), "pipelined": False,
                   "path": ("DistributedShard.apply" if sharded else "hb_apply via paper_2604_15765_b200.hermsim.apply")
                           + " + hs_state_upload/download_async"}
        L.hs_host_free(hbuf)  # before the CPU baseline: the reference needs the host RAM
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_from(cfg, n, m, psi=psi, strings=strings)

    for e in ev:
        L.hs_event_destroy(e)
    if rank != 0:
        return 0
    l2 = ("state %.3f GB per rank vs 126 MB L2: inputs larger than L2, no flush needed" % (S / 1e9))
    if S < 4 * 126e6:
        l2 = ("L2-ASSISTED: the %.0f MB state is about the 126 MB L2; consecutive ops alternate their sweep "
              "direction, so part of each op is served from L2 -- the roofline fraction is not an HBM-only "
              "number (ncu DRAM bytes per launch in roofline.traffic)" % (S / 1e6))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded rank-4 rho / Pauli-sum O of BASELINE.json shapes)",
        "config": {"workload": WORKLOADS[cfg], "config": cfg, "n": n, "m": m, "ops_per_step": nops,
                   "fused": ({"passes_per_step": npass, "note": "operation fusion (SURVEY 8f): value counts the "
                              "logical operations; reported separately from the per-operation metric"}
                             if fplan is not None else None),
                   "cuda_graph": bool(args.graph),
                   "stored_bytes_per_rank": S,
                   "parallelism": (f"sharded x{world} (XOR blocks, " + ("NCCL group exchange" if args.exchange else
                                   "peer-memory reads fused into the op kernels") +
                                   (", qubit remapping" if args.remap else "") + ")" if sharded else
                                   f"replicas x{world}" if world > 1 else "single GPU"),
                   "exchanges_per_step": (dshard.exchanges / max(1, args.warmup + args.steps + 1 + args.e2e_steps)
                                          if dshard is not None else 0),
                   "l2": l2},
        "achieved_hbm_gbs": sum(touched) * args.steps / (total_ms / 1e3) / 1e9,
        "touched_bytes_per_step": sum(touched),
        "effective_bandwidth_gbs_paper": S * nops * args.steps / (total_ms / 1e3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "pipe_kernel / gather_ws_kernel (csrc/engine.cu)",
                     "algorithmic_bytes_per_launch": per_launch_bytes,
                     "mean_launch_ms": mean_launch_ms, "min_launch_ms": min(launch_ms), "max_launch_ms": max(launch_ms),
                     "peak_source": peak_src, "traffic_source": traffic_src,
                     "scope": "rank 0's launches" if sharded else "all launches of one step"},
        "roofline_nvlink": roof_nv,
        "roofline_hbm_fp64": roof_mixed,
        "per_launch_ms": [round(x, 4) for x in launch_ms],
        "gpu_launches": launches,
        "host_wall_s": t_host,
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    line.update(result)
    print(json.dumps(line), flush=True)
    if dshard is not None:
        dshard.close()
    return 0


def stored_bytes(n: int, m: int = 5) -> int:
    G = (1 << n) >> m if n >= m else 1
    M = min(1 << m, 1 << n)
    return G * (G + 1) // 2 * M * M * 16


def cpu_sample_n(cfg: str, n: int, m: int, reserved: int = 0) -> int:
    """Largest n' <= n whose reference run fits this host's free RAM (where RAM is short,
    time at the largest feasible n and extrapolate x4 per qubit).  The input is built inside the
    reference's own buffer (one payload); its k = 3 path converts through three dense 4^n matrices
    (kernels.cpp:498-505)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available - reserved
    except Exception:  # pragma: no cover
        avail = 32 << 30
    budget = 0.85 * avail
    for k in range(n, 4, -1):
        dense3 = cfg in ("c3", "kraus")  # configs with k = 3 ops (the reference's dense round trip)
        need = 1.05 * stored_bytes(k, m) + (3 * 16 * (1 << (2 * k)) if dense3 else 0)
        # the dense k = 3 path also costs ~4^n time: keep a C3 sample within seconds per op
        if need <= budget and (not dense3 or k <= 13):
            return k
    return 5


def pipelined_e2e(args, H, L, nat, st, host0, S, n, m, nops, world, fplan, ops, opts):
    """End to end through the public API with consecutive steps overlapped, as a serving loop
    would run: up to --e2e-states device states and pinned host buffers; step k uploads its input into
    state k % B, applies the sequence and downloads the result, all on that state's stream, so
    uploads, compute and downloads of neighbouring steps overlap (PCIe is full duplex: ~91 GB/s
    both ways together on the box, tools/pcie_probe.cu).  Every step still moves S bytes
    host->device and S bytes device->host inside the timed region.  Returns None when not even a
    second state or pinned buffer fits (the serial loop is used then)."""
    cnt = st.element_count()
    states, bufs, pinned = [st], [host0], []
    try:
        import psutil
        host_total = psutil.virtual_memory().total
    except Exception:  # pragma: no cover
        host_total = 0
    for _ in range(max(0, args.e2e_states - 1)):  # up to e2e_states in flight when HBM and host memory allow
        if host_total and (len(bufs) + 1) * S > 0.75 * host_total:
            break  # keep a quarter of the host RAM free (pinned pages cannot be swapped)
        try:
            sx = H.TiledHermitian(n, m, device=st.device)
        except Exception:
            break
        hb = ctypes.c_void_p()
        if L.hs_host_alloc(ctypes.c_uint64(S), ctypes.byref(hb)) != 0:
            sx.free()
            break
        hx = np.ctypeslib.as_array(ctypes.cast(hb, ctypes.POINTER(ctypes.c_double)), shape=(2 * cnt,))
        hx[:] = host0
        states.append(sx)
        bufs.append(hx)
        pinned.append(hb)
    B = len(states)
    if B < 2:
        return None
    if fplan is not None:
        from paper_2604_15765_b200 import fusion

    def one(k):
        s, b = states[k % B], bufs[k % B]
        nat.check(L.hs_state_upload_async(s.handle, b.ctypes.data_as(nat.c_double_p), cnt))
        if fplan is not None:
            fusion.execute(s, fplan, opts)
        else:
            for spec, tg, _ in ops:
                H.apply(s, spec, tg, opts)
        nat.check(L.hs_state_download_async(s.handle, b.ctypes.data_as(nat.c_double_p), cnt))

    ev = [ctypes.c_void_p() for _ in range(1 + B)]
    for e in ev:
        nat.check(L.hs_event_create(ctypes.byref(e)))
    for k in range(B):  # warm-up round
        one(k)
    for s in states:
        s.synchronize()
    # enough steps that the pipeline fill (first upload alone) and drain (last download alone) are
    # a small part of the timed region (steady-state serving throughput): B = 3 -> 24 steps
    K = max(8 * B, args.e2e_steps)
    L.hs_event_record(ev[0], st.handle)  # all streams are idle: every later copy / kernel starts after it
    for k in range(K):
        one(k)
    for i, s in enumerate(states):
        L.hs_event_record(ev[1 + i], s.handle)
    for s in states:
        s.synchronize()
    total = 0.0
    for i in range(B):
        x = ctypes.c_float()
        nat.check(L.hs_event_elapsed_ms(ev[0], ev[1 + i], ctypes.byref(x)))
        total = max(total, x.value)
    for e in ev:
        L.hs_event_destroy(e)
    for s in states[1:]:
        s.free()
    for hb in pinned:
        L.hs_host_free(hb)
    ms = dist_max(total / K, world)
    return {"value": world * nops / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": S, "d2h_bytes_per_step": S,
            "ms_per_step": ms, "steps": K, "pipelined": True, "states_in_flight": B,
            "path": "hermsim.apply (or fusion.execute with --fuse) + hs_state_upload/download_async; consecutive "
                    "steps on different states overlap (upload k+1 || compute k || download k-1)"}


def cpu_baseline_from(cfg, n, m, psi=None, strings=None):
    """Reference CPU path on a bounded sample (about 10-30 s) of the same workload, rank 0 only:
    whole steps of the config when one fits in ~40 s (C0, C2: the full 12 / 32-op sequence), else
    blocks of 2 consecutive ops in stratified order within a 30 s budget."""
    try:
        from paper_2604_15765_b200 import harness as HS
        threads = os.cpu_count() or 1
        nc = cpu_sample_n(cfg, n, m)
        nops = len(HS.config_ops(cfg, nc))
        whole = cfg in ("c0", "c2") and nc == n
        fill = reference_fill(HS, cfg, nc, m, threads, psi=psi if nc == n else None,
                              strings=strings if nc == n else None)
        if whole:
            reps = 3 if cfg == "c0" else 1
            times, blocks, covered = run_reference_cpu(cfg, nc, m, fill, nops, reps, 1 if cfg == "c0" else 0, threads)
            ops_per_step = nops
        else:
            ops_per_step = 2
            times, blocks, covered = run_reference_cpu(cfg, nc, m, fill, ops_per_step, steps=64, warmup=0,
                                                       threads=threads, budget_s=30.0)
        t = float(np.mean(times))
        scale = 4.0 ** (n - nc)
        out = {"value": ops_per_step / t / scale, "unit": UNIT, "cores": threads, "kind": "reference",
               "sample": (f"{len(times)} full step(s) of {cfg} ({nops} ops)" if whole else
                          f"{len(times)} blocks of {ops_per_step} consecutive ops of {cfg} in stratified order "
                          f"(blocks {blocks})") + f" at n={nc} through hermsim::apply of the compiled reference "
                          "(oracle/_ref/libhermsim_ref.so), threads=nproc, input built in the reference's own buffer",
               "qubits_covered": covered}
        if nc != n:
            out["extrapolated_from_n"] = nc
            out["sample"] += f"; host RAM/time-bounded, extrapolated to n={n} by 4^(n-{nc}) (work grows 4x per qubit)"
        return out
    except Exception as e:  # the baseline is reported, never fatal
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference", "error": str(e)}


if __name__ == "__main__":
    sys.exit(main())
