"""Summarise an ncu --set full report (ncu -i REP --page raw --csv) into one line per launch:
duration, DRAM bytes, throughput, occupancy and pipe utilisation.  usage: ncu_summary.py REP"""
import csv
import io
import subprocess
import sys

WANT = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
        ("lts__t_sector_hit_rate.pct", "l2_hit_pct")]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {}
        for name, key in WANT:
            if name in hdr:
                i = hdr.index(name)
                d[key] = r[i] + ("" if key == "kernel" or not units[i] else f" {units[i]}")
        d["kernel"] = d["kernel"].split("(")[0]
        print("  ".join(f"{k}={v}" for k, v in d.items()))


if __name__ == "__main__":
    main(sys.argv[1])
