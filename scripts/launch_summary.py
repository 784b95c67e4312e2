"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.

usage: python scripts/launch_summary.py launches.csv [--skip-setup]
Prints per-kernel count, total, mean and share of the summed device time.  With
--skip-setup, launches before the first k_explicit launch of the timed loop are dropped
(setup kernels)."""
import collections
import csv
import re
import sys


def load(path):
    lines = open(path).read().splitlines()
    hi = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    out = []
    for row in csv.DictReader(lines[hi:]):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = row["Kernel Name"].split("(")[0]
        name = re.sub(r"<unnamed>::|\(anonymous namespace\)::|^void ", "", name)
        v = float(row["Metric Value"].replace(",", ""))
        u = row["Metric Unit"]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)
        out.append((name, v, row["Grid Size"], row["Block Size"]))
    return out


def summary(rows):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, v, *_ in rows:
        tot[n] += v
        cnt[n] += 1
    T = sum(tot.values())
    lines = [f"{'kernel':40s} {'n':>6s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k:40s} {cnt[k]:6d} {v:12.1f} {v / cnt[k]:10.2f} {v / T:7.3f}")
    lines.append(f"{'TOTAL':40s} {sum(cnt.values()):6d} {T:12.1f}")
    return "\n".join(lines)


if __name__ == "__main__":
    rows = load(sys.argv[1])
    if "--skip-setup" in sys.argv:
        # drop setup + startup: keep from the second k_explicit launch on
        idx = [i for i, r in enumerate(rows) if r[0].startswith(("k_explicit", "v2::k_exp3"))]
        if len(idx) > 1:
            rows = rows[idx[1]:]
    print(summary(rows))
