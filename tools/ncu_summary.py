#!/usr/bin/env python
"""Print the key ncu metrics of every kernel in a report (used for profiles/ summaries)."""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_red.sum",
        "lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "smsp__inst_executed.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]


def summary(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units = r[0], r[1]
    out = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = (row[hdr.index(k)], units[hdr.index(k)])
        stalls = {}
        for i, h in enumerate(hdr):
            m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio", h)
            if m:
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v > 0.2:
                    stalls[m.group(1)] = round(v, 2)
        d["stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        out.append(d)
    return out


if __name__ == "__main__":
    for d in summary(sys.argv[1]):
        print("=====", d.pop("kernel")[:60])
        st = d.pop("stalls")
        for k, (v, u) in d.items():
            print(f"  {k:60s} {v:>14s} {u}")
        print("  stalls:", st)
