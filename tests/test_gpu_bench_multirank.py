"""The bench's N > 1 code path (the driver's scaling run launches `torch.distributed.run
--nproc-per-node N bench.py --gpus N`), exercised functionally on ONE GPU: BENCH_FUNCTIONAL_ONE_GPU=1
puts every rank on GPU 0 with a gloo group, and the sharded peer mode orders the ranks by host
barriers, so no kernel waits on another (numbers from such a run are never measurements).  Checks
that every rank exits 0, rank 0 prints one JSON line with the sharded layout, the NVLink roofline
object and the reference arm's line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(nproc, args, timeout=900):
    env = dict(os.environ, BENCH_FUNCTIONAL_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(nproc)] + args
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg,n", [("c2", 12), ("c4", 13), ("c3", 11)])
def test_sharded_bench_two_ranks(cfg, n):
    line = _torchrun(2, ["--config", cfg, "--qubits", str(n), "--steps", "1", "--warmup", "3", "--no-cpu",
                         "--e2e-steps", "1"])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert "sharded x2" in line["config"]["parallelism"]
    assert line["roofline_nvlink"] is not None
    assert line["value"] > 0 and line["gpu_launches"] > 0
    print("MULTIRANK", cfg, n, line["value"], line["roofline_nvlink"].get("cross_shard_launches_per_step"))


def test_reference_arm_two_ranks():
    line = _torchrun(2, ["--impl", "reference", "--config", "c2", "--qubits", "10", "--steps", "1",
                         "--warmup", "1"])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"

