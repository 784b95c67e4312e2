"""Set up one BASELINE config on the GPU through the C ABI and report setup time, sizes
and per-step timings (diagnostics; not part of the bench contract).

usage: python scripts/probe_config.py CONFIG [STEPS]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import sc_inputs  # noqa: E402
import paper_2310_14712_b200 as pkg  # noqa: E402

cid = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = sc_inputs.get_config(cid)
stream = torch.cuda.Stream()
t0 = time.perf_counter()
s = pkg.from_config(cfg, f_t=sc_inputs.source_signal(cfg, steps + 10) if cfg["source"] else None,
                    stream=stream.cuda_stream)
setup = time.perf_counter() - t0
info = s.info
s.step(3)
s.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(stream):
    e0.record(stream)
    s.step(steps)
    e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
s.sync()
u = s.read()
prof = {}
for which, name in ((0, "explicit_ms"), (1, "celem_ms"), (2, "solve_ms")):
    with torch.cuda.stream(stream):
        e0.record(stream)
        s.profile(which, 10)
        e1.record(stream)
    torch.cuda.synchronize()
    prof[name] = e0.elapsed_time(e1) / 10
out = {"config": cid, "setup_s": setup, "ms_per_step": ms, "dof_steps_per_s": info["n_dof"] / (ms / 1e3),
       "u_norm": float(np.linalg.norm(u)), "mem_free_total": torch.cuda.mem_get_info(), "breakdown_ms": prof}
out.update({k: info[k] for k in info})
print(json.dumps(out, default=str))
