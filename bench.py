"""Benchmark of the Newmark IMEX time step (BASELINE.json metric: DOF-steps/s, FP64).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

* ours: the CUDA path through the C ABI (libsc.so).  W warm-up steps, then K steps timed
  with CUDA events on the library stream, barrier + synchronize on both sides, max over
  ranks.  With N > 1 ranks (torchrun) the ONE workload is slab-decomposed over the GPUs
  (NCCL exchange inside sc_step): value = n_dof * K / t, strong scaling.
* roofline: every sub-kernel of the step timed alone with CUDA events on the library
  stream (sc_profile); the dominant one (largest time) is reported against the measured
  HBM copy bandwidth with its algorithmic bytes (sc_query).
* e2e: one job through the public API with HOST buffers: sc_set_state(u0, v0 host) ->
  sc_step(K) -> sc_read(u host), copies inside the timed region.
* cpu_baseline / --impl reference: the CPU oracle (oracle/) as it stands, on the host
  cores, on a bounded sample of the same workload (its time loop, steps stated).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import sc_inputs  # noqa: E402

METRIC = "DOF-steps/sec (FP64) at 1/2/4/8 B200; achieved HBM GB/s vs peak"
UNIT = "DOF-steps/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, dev):
        self.dev = dev
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.1)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def sub_box(cfg, frac):
    """The same workload restricted to the corner sub-box [lo, lo + frac (hi - lo)]^d
    (same cell size, p, alpha, depth, dt; voids whose bounding sphere meets the box;
    the source kept only if it lies inside).  Used to bound the oracle's CPU time on the
    largest config; the sample is stated in the JSON line."""
    import copy
    c = copy.deepcopy(cfg)
    d = c["dim"]
    c["cells"] = [max(1, int(round(n * frac))) for n in cfg["cells"]]
    c["hi"] = [cfg["lo"][k] + (cfg["hi"][k] - cfg["lo"][k]) * c["cells"][k] / cfg["cells"][k] for k in range(d)]
    keep = []
    for v in cfg["voids"]:
        if v["kind"] != "ellipsoid":
            keep.append(v)
            continue
        A = np.array([[v["A"][0], v["A"][3], v["A"][4]], [v["A"][3], v["A"][1], v["A"][5]],
                      [v["A"][4], v["A"][5], v["A"][2]]])[:d, :d]
        R = 1.0 / np.sqrt(np.linalg.eigvalsh(A).min())
        ctr = np.array(v["c"][:d])
        near = np.clip(ctr, c["lo"], c["hi"])
        if np.linalg.norm(near - ctr) <= R:
            keep.append(v)
    c["voids"] = keep
    if c["source"] is not None and not all(c["lo"][k] <= c["source"]["x"][k] <= c["hi"][k] for k in range(d)):
        c["source"] = None
    c["name"] = cfg["name"] + f"-subbox{frac:g}"
    return c


def cpu_sample_cfg(cfg, frac=0.0625):
    """Config 5 (2.6e8 DOFs) is out of the oracle's reach in minutes: sample the corner
    sub-box of `frac` of the edge (default 1/16: 10^3 cells; same h, p, alpha, depth, dt,
    voids meeting the box).  The reference arm and cpu_baseline use the SAME sample."""
    if cfg["id"] == 5:
        n = int(round(cfg["cells"][0] * frac))
        return sub_box(cfg, frac), f"sub-box [0,{frac:g}]^3 ({n}^3 cells)"
    return cfg, "full size"


ORACLE_THREADS = 1   # the oracle's time loop (scipy sparse matvec + SuperLU solves) is serial


def oracle_sample(cfg, steps):
    """Time the oracle's IMEX loop (as it stands) on `steps` steps of `cfg`, with the BLAS /
    OpenMP pools limited to ORACLE_THREADS so that the reported core count is exact."""
    import oracle.assembly as OA
    from oracle.integrators import from_system, imex
    from oracle.run import initial_field
    n_dof_cells = np.prod(cfg["cells"]) * (cfg["p"] + 1) ** (2 * cfg["dim"])
    mode = "sparse" if n_dof_cells < 1.2e8 else "ebe"
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(ORACLE_THREADS)
    except Exception:
        lim = None
    try:
        t0 = time.perf_counter()
        sysm = OA.build_system(cfg, mode)
        t_setup = time.perf_counter() - t0
        pr = from_system(sysm)
        f_t = sc_inputs.source_signal(cfg, steps + 1)
        u0 = initial_field(cfg, sysm)
        t0 = time.perf_counter()
        imex(pr, cfg["dt"], steps, f_t, u0, None)
        t = time.perf_counter() - t0
    finally:
        if lim is not None:
            lim.restore_original_limits()
    return sysm.n_dof * steps / t, t, t_setup, sysm.n_dof, mode


def _cpu_line(args, steps):
    cfg = sc_inputs.get_config(args.config)
    scfg, what = cpu_sample_cfg(cfg)
    value, t, t_setup, n_dof, mode = oracle_sample(scfg, steps)
    sample = (f"config {args.config} {what} ({n_dof} DOFs, {mode} assembly), oracle IMEX time loop of "
              f"{steps} steps ({t:.2f} s; setup {t_setup:.1f} s untimed), {ORACLE_THREADS} thread")
    return {"value": value, "unit": UNIT, "cores": ORACLE_THREADS, "kind": "oracle", "sample": sample}, t


def run_reference(args, rank):
    if rank != 0:
        return 0
    cfg = sc_inputs.get_config(args.config)
    # bounded sample: the oracle's IMEX time loop (setup untimed), ref_steps oracle steps per
    # timed step on the same sample as cpu_baseline (config 5: the corner 10^3-cell sub-box,
    # ~0.04 s per oracle step), so that the whole run stays within a few minutes
    nsteps = max(1, args.steps) * max(1, args.ref_steps)
    cpu, t = _cpu_line(args, nsteps)
    value = cpu["value"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / nsteps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_dict(cfg), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _config_dict(cfg):
    """The workload descriptor (identical for both arms; sizes found by the setup are reported
    outside it, under "problem")."""
    return {"workload": f"config{cfg['id']}: {cfg['name']}", "dim": cfg["dim"], "cells": cfg["cells"],
            "p": cfg["p"], "n_voids": len(cfg["voids"]), "alpha": cfg["alpha"], "tree_depth": cfg["tree_depth"],
            "dt": cfg["dt"], "steps_per_job": "--steps", "source": "Ricker point source" if cfg["source"] else "none",
            "l2": "per-step working set larger than L2 (no flush)" if cfg["id"] in (4, 5) else
                  "L2-resident working set (no flush)"}


def _relaunch(args):
    """--gpus N > 1 without a torchrun environment: launch N ranks (one per GPU) of this script
    under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    import socket
    import torch
    if torch.cuda.device_count() < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but {torch.cuda.device_count()} CUDA devices visible"}),
              flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-steps", type=int, default=1, help="oracle steps per timed step (reference arm)")
    ap.add_argument("--cpu-steps", type=int, default=300, help="oracle steps for cpu_baseline")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch(args)
    if world != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)

    import torch
    import torch.distributed as dist
    import paper_2310_14712_b200 as pkg
    torch.cuda.set_device(local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(pkg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    W, K = max(3, args.warmup), args.steps
    cfg = sc_inputs.get_config(args.config)
    f_t = sc_inputs.source_signal(cfg, W + K + 2) if cfg["source"] else None
    stream = torch.cuda.Stream()
    t0 = time.perf_counter()
    s = pkg.from_config(cfg, f_t=f_t, stream=stream.cuda_stream, device=local, rank=rank, world=world,
                        nccl_id=nccl_id)
    setup_s = time.perf_counter() - t0
    info = s.info
    n_dof = info["n_dof"]
    s.step(W)
    s.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    clk.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        s.step(K)
        e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    s.sync()   # raises on a non-finite state
    t_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = n_dof * K / (t_ms / 1e3)   # the whole (decomposed) workload
    # ---- per-kernel timings (each sub-kernel timed alone with CUDA events on the library
    # stream, sc_profile) and the roofline of the dominant one (largest time per step)
    peak, peak_kind = _peaks()
    kern = {"explicit": (0, info["bytes_explicit_per_step"], "k_explicit (a1)+(a2), tensor-d DOFs"),
            "celem": (1, info["bytes_celem_per_step"], "k_celem_sym + k_celem_ref (a3)+(a4) c-element products"),
            "solve": (2, info["bytes_solve_per_step"], "k_solve (a5) persistent supernodal solve")}
    breakdown = {}
    for name, (which, nbytes, _) in kern.items():
        if which in (1, 2) and info["n_c"] == 0:
            continue
        nprof = 30
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            s.profile(which, nprof)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / nprof
        breakdown[name] = {"ms": ms, "algorithmic_bytes": nbytes, "GBps": nbytes / (ms / 1e3) / 1e9,
                           "frac": nbytes / (ms / 1e3) / 1e9 / peak}
    dom = max(breakdown, key=lambda k: breakdown[k]["ms"])
    bd = breakdown[dom]
    # measured DRAM traffic per launch of that kernel from the committed ncu --set full capture
    # of the same workload (scripts/ncu_traffic.py), when there is one
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_config{cfg['id']}.json")
    kname = {"explicit": "v2::k_exp3" if cfg["dim"] == 3 else f"k_explicit_{cfg['dim']}d",
             "celem": "k_celem", "solve": "k_solve"}[dom]
    if world == 1 and os.path.exists(tpath):
        tj = json.load(open(tpath))
        if kname in tj:
            traffic, traffic_src = tj[kname]["bytes"], tj[kname]["report"]
    roof = {"kernel": kern[dom][2], "bound": "hbm", "achieved": bd["GBps"], "peak": peak, "unit": "GB/s",
            "frac": bd["frac"], "traffic": traffic, "traffic_source": traffic_src, "peak_kind": peak_kind,
            "kernel_ms": bd["ms"], "share_of_step": bd["ms"] / (t_ms / K),
            "algorithmic_bytes": bd["algorithmic_bytes"]}
    # ---- e2e through the public API with host buffers (pinned): the initial state goes
    # host -> device, K steps, the final displacement comes back device -> host
    u0t = torch.zeros(n_dof, dtype=torch.float64).pin_memory()
    if cfg.get("u0") == "gaussian_pulse":
        u0t.copy_(torch.from_numpy(sc_inputs.gaussian_pulse(s.dof_coords()[:, 0])))
    uht = torch.empty(n_dof, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with torch.cuda.stream(stream):
        e0.record(stream)
        s.set_state(u0t.numpy(), None)   # v0 = 0 (every config starts at rest)
        s.step(K)
        s.read(uht.numpy())
        e1.record(stream)
    torch.cuda.synchronize()
    t_e2e = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([t_e2e], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e = {"value": n_dof * K / (t_e2e / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": 8.0 * n_dof / K, "d2h_bytes_per_step": 8.0 * n_dof / K,
           "job": f"sc_set_state(u0 pinned host, v0 = 0) + sc_step({K}) + sc_read(u pinned host)"}
    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu, _ = _cpu_line(args, args.cpu_steps)
        except Exception as ex:  # report, do not fail the bench
            cpu = {"value": None, "unit": UNIT, "cores": ORACLE_THREADS, "kind": "oracle", "sample": f"failed: {ex}"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "config": _config_dict(cfg),
                "problem": {"n_dof": n_dof, "n_c": info["n_c"], "n_d": info["n_d"], "cells_cut": info["cells_cut"],
                            "n_components": info["n_components"], "n_supernodes": info["n_supernodes"],
                            "nnz_factor": info["nnz_factor"], "factor_height": info["factor_height"],
                            "kernels_per_step": info["kernels_per_step"],
                            "parallelism": (f"z-slabs over {world} GPUs, NCCL exchange" if world > 1 else "1 GPU"),
                            "halo_values_per_step": info["halo_send"], "n_c_rank0": info["n_c_local"]},
                "roofline": roof, "kernels": breakdown, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
                "gpu_launches": int(info["kernels_per_step"]) * K,
                "step_bytes_algorithmic": info["bytes_per_step"],
                "step_achieved_GBps": info["bytes_per_step"] / (t_ms / K / 1e3) / 1e9,
                "setup_s": setup_s}
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
