"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of each kernel in an
ncu --set full report -> JSON {kernel: {"bytes": B, "launches": n, "report": path}} that
bench.py reads for roofline.traffic.  usage: ncu_traffic.py REPORT OUT.json [WORKLOAD]"""
import csv
import io
import json
import subprocess
import sys


def main(rep, out, workload=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        name = name.split("<")[0]
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(r[i]) * scale[units[i]]
        a = acc.setdefault(name, {"bytes": 0.0, "launches": 0})
        a["bytes"] += b
        a["launches"] += 1
    res = {k: {"bytes": v["bytes"] / v["launches"], "launches": v["launches"], "report": rep, "workload": workload}
           for k, v in acc.items()}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
