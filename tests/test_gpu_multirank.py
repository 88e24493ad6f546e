"""The sharded bench flow end to end with several ranks on the one GPU the
test box has: torchrun, process group over gloo (NCCL refuses two ranks on one
device), weak and strong scaling.  Each rank runs bench.py's correctness guard
(its owned rows of y against cuSPARSE, boundary fix-ups included) before any
timing; the timings of ranks sharing a GPU mean nothing and are not checked.
No kernel waits on another rank: the exchange is host-mediated."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("n,workload,scaling,iterative", [(2, "lap5_1000", "weak", False),
                                                          (3, "lap5_1000", "strong", False),
                                                          (4, "lap5_1000", "weak", False),
                                                          (3, "lap5_1000", "weak", True)])
def test_bench_sharded_on_one_gpu(n, workload, scaling, iterative):
    env = dict(os.environ, CSR5G_DIST_BACKEND="gloo", CSR5G_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
           "--gpus", str(n), "--steps", "3", "--warmup", "3", "--workload", workload,
           "--scaling", scaling] + (["--iterative"] if iterative else [])
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 prints one line
    d = lines[0]
    assert d["n_gpus"] == n and d["scaling"] == scaling
    assert d["correctness_max_rel_err"] <= 1e-12
    m1 = 1000 * 1000
    assert d["config"]["m"] == (m1 * n if scaling == "weak" else m1)


@pytest.mark.gpu
@pytest.mark.parametrize("iterative", [False, True])
def test_bench_two_distinct_gpus(iterative):
    """The real thing, on a box with two or more GPUs: one rank per GPU over
    NCCL, the boundary partials and (iterative) the fused y -> x stores over
    NVLink P2P, every rank's correctness guard before timing.  Skipped on the
    one-GPU test box (the round's GPU tier has one device)."""
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip(f"needs two GPUs, this box has {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "rmat24",
           "--scaling", "strong"] + (["--iterative"] if iterative else [])
    r = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["correctness_max_rel_err"] <= 1e-12
    assert d["value"] > 0 and d["gpu_launches"] >= 3
