"""Attribute an ncu SASS source page to CUDA source lines.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTRING [--lib paper_2501_17779_b200/libcurvalign_cuda.so]

Joins `ncu --page source --print-source sass` (per-instruction warp-stall
samples and executed instructions) with `nvdisasm -gi` line info of the same
cubin (the library is compiled with -lineinfo) and prints the hottest
file:line entries.
"""
from __future__ import annotations

import argparse
import collections
import csv
import glob
import io
import os
import re
import subprocess
import tempfile


def sass_page(report, kernel):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    recs = []
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr):
            continue
        recs.append(dict(zip(hdr, r)))
    return recs


def line_map(lib, kernel, recs=None):
    """addr -> file:line for the function whose SASS matches the ncu page."""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    maps, ops = {}, {}
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
        cur_fn, loc, fresh = None, None, True
        for ln in txt.splitlines():
            f = re.match(r"\s*\.text\.(\S+):", ln)
            if f:
                cur_fn = f.group(1)
                if kernel in cur_fn:
                    maps.setdefault(cur_fn, {})
                    ops.setdefault(cur_fn, [])
                continue
            g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if g:
                if fresh:  # the first annotation after an instruction is the innermost frame
                    loc = f"{os.path.basename(g.group(1))}:{g.group(2)}"
                    fresh = False
                continue
            a = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if a:
                fresh = True
                if cur_fn and kernel in cur_fn:
                    maps[cur_fn][int(a.group(1), 16)] = loc
                    ops[cur_fn].append(a.group(2).split()[0])
    if recs is None or len(maps) <= 1:
        return next(iter(maps.values()), {})
    want = [r["Source"].split()[0] for r in recs]
    best = max(maps, key=lambda fn: (len(ops[fn]) == len(want), sum(a == b for a, b in zip(ops[fn], want))))
    return maps[best]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--lib", default="paper_2501_17779_b200/libcurvalign_cuda.so")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--op", default=None, help="only SASS opcodes matching this regex (e.g. 'MOV')")
    a = ap.parse_args()
    recs = sass_page(a.report, a.kernel)
    lm = line_map(a.lib, a.kernel.split("::")[-1], recs)
    samp = collections.Counter()
    inst = collections.Counter()
    tot_s = tot_i = 0
    base = int(recs[0]["Address"], 16) if recs else 0
    for r in recs:
        if a.op and not re.search(a.op, r["Source"].split(" ")[0] if not r["Source"].lstrip().startswith("@")
                                  else r["Source"].split()[1]):
            continue
        addr = int(r["Address"], 16) - base
        loc = lm.get(addr, "?")
        s = int(float(r.get("Warp Stall Sampling (All Samples)", "0") or 0))
        i = int(float(r.get("Instructions Executed", "0") or 0))
        samp[loc] += s
        inst[loc] += i
        tot_s += s
        tot_i += i
    print(f"{'samples%':>9} {'inst%':>7}  location")
    for loc, s in samp.most_common(a.top):
        print(f"{100 * s / max(tot_s, 1):9.2f} {100 * inst[loc] / max(tot_i, 1):7.2f}  {loc}")


if __name__ == "__main__":
    main()
