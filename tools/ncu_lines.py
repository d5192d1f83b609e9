#!/usr/bin/env python
"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: tools/ncu_lines.py <report.ncu-rep> <cubin-or-.so> <mangled kernel name> [top]
Joins `ncu --page source --csv` (SASS, per-instruction samples) with `nvdisasm -g` line
info by instruction offset (requires -lineinfo).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(lib, kernel):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    out = {}
    for f in os.listdir(d):
        if not f.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True, text=True).stdout
        if kernel not in txt:
            continue
        in_fn, cur = False, None
        for line in txt.splitlines():
            if line.startswith("//---") and ".text." in line:
                in_fn = line.strip().endswith(kernel + " --------------------------") or (".text." + kernel) in line
                continue
            if not in_fn:
                continue
            m = re.search(r'line (\d+)', line)
            if "//## File" in line and m:
                cur = (os.path.basename(line.split('"')[1]), int(m.group(1)))
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
            if m and cur:
                out[int(m.group(1), 16)] = cur
    return out


def kernel_rows(rep, kernel):
    """rows (kernel line, header, data...) of the first kernel block whose demangled name
    contains the unmangled kernel name."""
    csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(csvtxt)))
    short = re.sub(r"^_ZN\d+\w+?\d+", "", kernel)
    m = re.match(r"_ZN(\d+)(\w+)", kernel)
    want = None
    if m:  # _ZN4memk8k_pointsI... -> "k_points"
        rest = kernel[len("_ZN"):]
        names = []
        while rest and rest[0].isdigit():
            n = int(re.match(r"\d+", rest).group(0))
            rest = rest[len(str(n)):]
            names.append(rest[:n])
            rest = rest[n:]
        want = names[-1] if names else None
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r]
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    for b in blocks:
        if want is None or want in b[0][1]:
            return b
    return blocks[0]


def main():
    rep, lib, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    col = sys.argv[5] if len(sys.argv) > 5 else "Warp Stall Sampling (All Samples)"
    lines = sass_lines(lib, kernel)
    rows = kernel_rows(rep, kernel)
    hdr = rows[1]
    si = hdr.index(col)
    data = rows[2:]
    base = int(data[0][0], 16)
    agg = collections.Counter()
    tot = 0
    for r in data:
        n = int(float(r[si] or 0))
        tot += n
        agg[lines.get(int(r[0], 16) - base, ("?", 0))] += n
    src = {}
    for (f, ln), n in agg.most_common(top):
        path = os.path.join(os.path.dirname(lib), "csrc", f)
        if f not in src and os.path.exists(path):
            src[f] = open(path).read().splitlines()
        text = src.get(f, [""] * (ln + 1))[ln - 1].strip() if ln else ""
        print(f"{n:7d} {100.0 * n / tot:5.1f}%  {f}:{ln:<5d} {text[:90]}")


if __name__ == "__main__":
    main()


def groups(rep, lib, kernel, ranges):
    """sum samples over named (file, first, last) line ranges."""
    lines = sass_lines(lib, kernel)
    rows = kernel_rows(rep, kernel)
    hdr = rows[1]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    data = rows[2:]
    base = int(data[0][0], 16)
    agg = collections.Counter()
    tot = 0
    for r in data:
        n = int(r[si] or 0)
        tot += n
        f, ln = lines.get(int(r[0], 16) - base, ("?", 0))
        name = "other"
        for nm, (ff, a, b) in ranges.items():
            if f == ff and a <= ln <= b:
                name = nm
                break
        agg[name] += n
    return {k: round(100.0 * v / tot, 1) for k, v in agg.most_common()}
