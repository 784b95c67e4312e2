"""Time the persistent supernodal solve (a5) of one config under solve-layout variants and,
with SC_TRACE, analyse one launch's item timeline (diagnostics, not part of the bench).

usage: python scripts/probe_solve.py CONFIG [TILE:FUSE ...]     (runs each variant in a subprocess)
       python scripts/probe_solve.py --analyse TRACE_FILE"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def analyse(path):
    raw = open(path, "rb").read()
    n_items, n_sn = np.frombuffer(raw[:8], np.int32)
    off = 8
    items = np.frombuffer(raw[off:off + 80 * n_items], np.int32).reshape(n_items, 20)
    off += 80 * n_items
    tr5 = np.frombuffer(raw[off:off + 40 * n_items], np.uint64).reshape(n_items, 5).astype(np.int64)
    off += 40 * n_items
    tr = tr5[:, [1, 2, 4]]   # item known, gathered, done
    wrp = np.frombuffer(raw[off:off + 12 * n_sn], np.int32).reshape(3, n_sn)
    w, r, parent = wrp
    t0 = tr[:, 0].min()
    tr = tr - t0
    height = np.zeros(n_sn, np.int64)
    for s in range(n_sn):   # children precede parents in the numbering used by the factor
        if parent[s] >= 0:
            height[parent[s]] = max(height[parent[s]], height[s] + 1)
    ph = items[:, 0]
    fused = items[:, 3] == 1   # single-tile groups
    d = np.diff(tr5 - tr5[:, :1], axis=1) / 1e3
    out = {"stage_us_median": {k: round(float(np.median(d[:, i])), 2) for i, k in
                               enumerate(["claim->item", "item->gathered", "gathered->staged", "staged->done"])},
           "stage_us_p90": {k: round(float(np.percentile(d[:, i], 90)), 2) for i, k in
                            enumerate(["claim->item", "item->gathered", "gathered->staged", "staged->done"])},
           "span_us": float(tr[:, 2].max() / 1e3), "n_items": int(n_items),
           "fused_work_us_mean": float((tr[fused, 2] - tr[fused, 1]).mean() / 1e3) if fused.any() else None,
           "tiled_work_us_mean": float((tr[~fused, 2] - tr[~fused, 1]).mean() / 1e3) if (~fused).any() else None,
           "wait_us_mean": float((tr[:, 1] - tr[:, 0]).mean() / 1e3)}
    # stage medians per (phase, single-tile) group
    groups = {}
    for p_ in (0, 1):
        for fz in (True, False):
            m = (ph == p_) & (fused == fz)
            if m.any():
                groups[("F" if p_ == 0 else "B") + ("-fused" if fz else "-tiled")] = [
                    int(m.sum())] + [round(float(np.median(d[m, i])), 2) for i in range(4)]
    out["stage_median_by_group"] = groups
    levels = []
    H = int(height.max()) + 1
    for p_ in (0, 1):
        for h in (range(H) if p_ == 0 else range(H - 1, -1, -1)):
            m = (ph == p_) & (height[items[:, 1]] == h)
            if not m.any():
                continue
            nbytes = 8 * (items[m, 7].astype(np.int64) * items[m, 9]).sum()
            levels.append({"phase": "F" if p_ == 0 else "B", "h": h, "start": round(float(tr[m, 1].min() / 1e3), 1),
                           "end": round(float(tr[m, 2].max() / 1e3), 1), "items": int(m.sum()),
                           "fused": int((m & fused).sum()), "MB": round(float(nbytes) / 1e6, 1),
                           "max_work_us": round(float((tr[m, 2] - tr[m, 1]).max() / 1e3), 2)})
    out["levels"] = levels
    print(json.dumps(out))


def run_variant(cid, tile, fuse, trace):
    env = dict(os.environ, SC_SOLVE_TILE=str(tile), SC_FUSE_ENTRIES=str(fuse))
    if trace:
        env["SC_TRACE"] = trace
    code = f"""
import sys, json, torch
sys.path.insert(0, {ROOT!r})
import sc_inputs, paper_2310_14712_b200 as pkg
cfg = sc_inputs.get_config({cid})
st = torch.cuda.Stream()
s = pkg.from_config(cfg, f_t=sc_inputs.source_signal(cfg, 64) if cfg['source'] else None, stream=st.cuda_stream)
s.step(5); s.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st); s.profile(2, 50); e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
s.profile(2, 1); s.sync()
print(json.dumps({{"tile": {tile}, "fuse": {fuse}, "solve_ms": ms, "nnz": s.info["nnz_factor"]}}))
s.close()
"""
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--analyse":
        analyse(sys.argv[2])
    else:
        cid = int(sys.argv[1])
        variants = sys.argv[2:] or ["256:16384"]
        for k, v in enumerate(variants):
            tile, fuse = map(int, v.split(":"))
            tp = f"/tmp/trace_c{cid}_{tile}_{fuse}.bin"
            run_variant(cid, tile, fuse, tp)
            if os.path.exists(tp):
                analyse(tp)
