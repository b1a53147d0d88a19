"""Per-source-line table of an ncu report: executed instructions, stall samples by reason and
excess shared-memory wavefronts (bank conflicts).

    python tools/ncu_lines2.py REPORT KERNEL [--sort stall_short_sb] [--top 40] [--lib ...]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines as nl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("kernel")
ap.add_argument("--sort", default="Warp Stall Sampling (All Samples)")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--lib", default="paper_2501_17779_b200/libcurvalign_cuda.so")
a = ap.parse_args()
recs = nl.sass_page(a.report, a.kernel)
lm = nl.line_map(a.lib, a.kernel.split("::")[-1], recs)
base = int(recs[0]["Address"], 16)
cols = ["Instructions Executed", "Warp Stall Sampling (All Samples)", "stall_short_sb", "stall_long_sb", "stall_wait",
        "stall_barrier", "stall_no_inst", "stall_mio", "L1 Wavefronts Shared Excessive"]
agg = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for r in recs:
    loc = lm.get(int(r["Address"], 16) - base, "?")
    for c in cols:
        x = float((r.get(c) or "0").replace(",", "") or 0)
        agg[loc][c] += x
        tot[c] += x
short = ["inst", "samp", "short", "long", "wait", "bar", "noinst", "mio", "xsWF"]
print(f"{'location':26s} " + " ".join(f"{s:>7s}" for s in short) + "   (% of kernel totals)")
for loc, c in sorted(agg.items(), key=lambda kv: -kv[1][a.sort])[: a.top]:
    print(f"{loc:26s} " + " ".join(f"{100 * c[k] / max(tot[k], 1):7.2f}" for k in cols))
print("totals:", {s: int(tot[c]) for s, c in zip(short, cols)})
