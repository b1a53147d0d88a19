"""Aggregate an ncu report's SASS source page by opcode (executed warp instructions).

    python tools/sass_mix.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
ci, cs, ct, cp = (h.index("Instructions Executed"), h.index("Source"), h.index("Thread Instructions Executed"),
                  h.index("Predicated-On Thread Instructions Executed"))
cnt = collections.Counter()
thr = collections.Counter()
tot = 0
for r in rows[hdr + 1:]:
    if len(r) <= ci or not r[ci].strip():
        continue
    src = r[cs].strip()
    parts = src.split()
    if not parts:
        continue
    op = parts[0]
    if op.startswith("@"):
        op = parts[1]
    base = op.split(".")[0]
    n = int(float(r[ci]))
    cnt[base] += n
    thr[base] += int(float(r[cp]))
    tot += n
print(f"total warp inst {tot:,}")
for op, n in cnt.most_common(top):
    print(f"{op:10s} {n:14,d} {100.0 * n / tot:6.2f}%  active lanes {thr[op] / max(n, 1):5.1f}")
