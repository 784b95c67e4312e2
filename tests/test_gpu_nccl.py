"""The NCCL transport of the slab decomposition on >= 2 GPUs: one process per
GPU (tests/nccl_worker.py under torch.distributed.run on 127.0.0.1), the exchange inside
sc_step, the collective sc_read.  Config 2 is checked against the oracle (1e-10) and config 5
against the single-GPU run (bit-identical: every rank applies the same per-node arithmetic).
Skipped with fewer than 2 CUDA devices (the in-process multi-rank path is covered on one GPU
by tests/test_gpu_multirank.py)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import sc_inputs
from oracle.run import run_config

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 CUDA devices")
    from paper_2310_14712_b200.build import build
    build()
    import paper_2310_14712_b200 as p
    p.load_library()
    return p


def _run(world, cid, steps, tmp_path):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / f"u_{cid}_{world}.npy")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "nccl_worker.py"),
           str(cid), str(steps), out]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return np.load(out)


def test_nccl_config2_vs_oracle(pkg, tmp_path):
    steps = 400
    u = _run(2, 2, steps, tmp_path)
    ref, _ = run_config(sc_inputs.get_config(2), steps=steps)
    err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
    assert err <= 1e-10, err


def test_nccl_config5_matches_one_gpu(pkg, tmp_path):
    import torch
    world = min(4, torch.cuda.device_count())
    steps = 6
    u = _run(world, 5, steps, tmp_path)
    s = pkg.from_config(sc_inputs.get_config(5))
    s.step(steps)
    u1 = s.read()
    s.close()
    assert np.array_equal(u, u1)
