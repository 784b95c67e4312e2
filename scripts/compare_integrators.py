"""The paper's efficiency comparison (Table tab:times3D P:1473-1479) on the GPU: Newmark
IMEX at the config's dt (0.9 x the uncut cell-wise critical step) vs CDM on the HRZ-lumped and
on the consistent SCM at 0.9 x their own critical steps (device power iteration), and (2D
configs) trapezoidal Newmark on all DOFs at the IMEX dt.  Reports ms/step and simulated time
per wall second (dt / step time).  usage: compare_integrators.py CONFIG [STEPS]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import sc_inputs  # noqa: E402
import paper_2310_14712_b200 as pkg  # noqa: E402


def timed(cfg, steps, stream):
    s = pkg.from_config(cfg, f_t=sc_inputs.source_signal(cfg, 4 * steps + 64) if cfg["source"] else None,
                        stream=stream.cuda_stream)
    s.step(5)
    s.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        s.step(steps)
        e1.record(stream)
    torch.cuda.synchronize()
    s.sync()
    ms = e0.elapsed_time(e1) / steps
    return s, ms


cid = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
st = torch.cuda.Stream()
cfg = sc_inputs.get_config(cid)
out = {"config": cid, "n_dof": None}
s, ms = timed(cfg, steps, st)
_, dt_imex_crit = s.estimate_dt(3000)
out["n_dof"] = s.info["n_dof"]
s.close()
out["imex"] = {"dt": cfg["dt"], "dt_crit_est": dt_imex_crit, "ms_per_step": ms,
               "sim_time_per_wall_s": cfg["dt"] / (ms / 1e3)}
for name in ("cdm_hrz", "cdm_consistent"):
    h = dict(cfg)
    h["integrator"] = name
    s = pkg.from_config(h)
    _, dtc = s.estimate_dt(3000)
    s.close()
    h["dt"] = 0.9 * dtc
    s, ms = timed(h, steps, st)
    s.close()
    out[name] = {"dt": h["dt"], "dt_crit_est": dtc, "ms_per_step": ms, "sim_time_per_wall_s": h["dt"] / (ms / 1e3)}
if cfg["dim"] == 2:
    h = dict(cfg)
    h["integrator"] = "trapezoidal"
    s, ms = timed(h, steps, st)
    s.close()
    out["trapezoidal"] = {"dt": h["dt"], "ms_per_step": ms, "sim_time_per_wall_s": h["dt"] / (ms / 1e3)}
out["imex_speedup_at_equal_simulated_time"] = {
    k: out["imex"]["sim_time_per_wall_s"] / out[k]["sim_time_per_wall_s"]
    for k in ("cdm_hrz", "cdm_consistent", "trapezoidal") if k in out}
print(json.dumps(out))
