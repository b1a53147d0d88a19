"""Summarise one kernel of an `ncu --set full` report into profiles/*.json.

    python tools/ncu_summary.py REPORT.ncu-rep KERNEL_REGEX OUT.json [--round r2] [--algorithmic-bytes B]

Reads `ncu -i REPORT --page raw --csv` and keeps the metrics the bench and
DESIGN.md quote: duration, DRAM bytes, FP64 pipe, issue, occupancy, stall
breakdown per issued instruction and shared-memory bank conflicts.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess

KEEP = {
    "gpu__time_duration.sum": "gpu__time_duration_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "sm__pipe_fp64_cycles_active_pct",
    "smsp__inst_executed.sum": "smsp__inst_executed_sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__maximum_warps_per_active_cycle_pct": "theoretical_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__shared_mem_per_block_dynamic": "dynamic_smem_per_block_KB",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__inst_executed.avg.per_cycle_active": "executed_ipc_active",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("out")
    ap.add_argument("--round", default="")
    ap.add_argument("--command", default="")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv", "-k", f"regex:{a.kernel}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name"), "round": a.round, "command": a.command}
    for k, name in KEEP.items():
        if k in d:
            v = num(d[k])
            unit = u.get(k, "")
            if name.endswith("_MB") and isinstance(v, float):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0,
                         "GB": 1e3}.get(unit, 1.0)
            if name == "gpu__time_duration_us" and isinstance(v, float):
                v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
            if name == "dynamic_smem_per_block_KB" and isinstance(v, float):
                v = v * {"byte": 1e-3, "Kbyte": 1.0}.get(unit, 1.0)
            out[name] = v
    if "dram_read_MB" in out and "dram_write_MB" in out:
        out["dram_bytes_per_launch"] = int(round((out["dram_read_MB"] + out["dram_write_MB"]) * 1e6))
    if a.algorithmic_bytes:
        out["algorithmic_bytes_per_launch"] = int(a.algorithmic_bytes)
    # FP64 instruction work of the launch (thread-level DADD + DMUL + DFMA, each
    # one pipe op) and the time it needs at the SMs' FP64 op rate: the compute
    # floor of the kernel as written, next to its HBM floor.
    ops = [num(d.get(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed", "x"))
           for o in ("dadd", "dmul", "dfma")]
    cyc = num(d.get("sm__cycles_elapsed.avg", "x"))
    peak = num(d.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained", "x"))
    if all(isinstance(x, float) for x in ops + [cyc, peak]) and peak > 0:
        total = sum(ops) * cyc
        out["fp64_thread_ops_per_launch"] = int(round(total))
        out["fp64_op_floor_cycles"] = int(round(total / peak))
        out["fp64_op_utilisation_pct"] = 100.0 * sum(ops) / peak
    stalls = {}
    for k in hdr:
        m = re.fullmatch(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", k)
        if m and num(d[k]) not in ("", 0.0):
            stalls[m.group(1)] = num(d[k])
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
