"""P13: the partitioned IMEX of oracle/partition.py, run by 2 processes over
torch.distributed gloo (CPU), reproduces the single-process oracle.  Voids straddle the slab
boundary, so the component ownership and the exchange are exercised."""
import os
import socket

import numpy as np
import pytest

import sc_inputs
from oracle.assembly import build_system
from oracle.integrators import from_system, imex
from oracle.spectra import dt_crit_uncut

CFG = sc_inputs.small_config(2, [10, 12], 3, voids=[
    {"kind": "ellipsoid", "c": [0.4, 0.55, 0.0], "A": [60.0, 50.0, 0.0, 6.0, 0.0, 0.0]},
    {"kind": "ellipsoid", "c": [0.8, 0.15, 0.0], "A": [400.0, 400.0, 0.0, 0.0, 0.0, 0.0]}],
    depth=3, steps=60, source={"x": [0.2, 0.7, 0.0], "f0": 5.0})
CFG["dt"] = 0.9 * dt_crit_uncut(2, 3, 1.0 / 12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from oracle.partition import imex_partitioned, owners
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sysm = build_system(CFG, "sparse")
    pr = from_system(sysm)
    nl = [CFG["cells"][k] * CFG["p"] + 1 for k in range(2)]
    own = owners(pr, sysm.cl.lattice_index, nl, CFG["p"], CFG["cells"][-1], world)

    def allgather(vec):
        t = torch.from_numpy(vec)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.numpy() for p in parts]

    f_t = sc_inputs.source_signal(CFG, CFG["steps"] + 1)
    u = imex_partitioned(pr, CFG["dt"], CFG["steps"], f_t, np.zeros(pr.n), own, rank, world, allgather)
    np.save(os.path.join(out, f"u{rank}.npy"), u)
    np.save(os.path.join(out, f"own{rank}.npy"), own)
    dist.destroy_process_group()


def test_two_rank_gloo_partition_matches_oracle(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    sysm = build_system(CFG, "sparse")
    pr = from_system(sysm)
    f_t = sc_inputs.source_signal(CFG, CFG["steps"] + 1)
    ref = imex(pr, CFG["dt"], CFG["steps"], f_t, np.zeros(pr.n))
    u0, u1 = np.load(tmp_path / "u0.npy"), np.load(tmp_path / "u1.npy")
    own = np.load(tmp_path / "own0.npy")
    assert 0 < (own == 1).sum() < len(own)                      # both ranks own DOFs
    assert set(own[pr.I_c].tolist()) == {0, 1}                   # each rank solves a component
    assert np.array_equal(u0, u1)                                # ranks agree exactly
    err = np.linalg.norm(u0 - ref) / np.linalg.norm(ref)
    assert err < 1e-11, err
