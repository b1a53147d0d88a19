"""One-screen summary of an ncu --set full report: time, issue, occupancy, FP64 pipe, stalls,
instruction mix by class and per source region.

    python tools/ncu_brief.py report.ncu-rep [kernel_regex]
"""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
args = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", f"regex:{kre}"] if kre else [])
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
def g(k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return float("nan")
keys = [("gpu__time_duration.sum", "time ns"), ("smsp__inst_executed.sum", "warp inst"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst pipe %"),
        ("launch__registers_per_thread", "regs"), ("launch__shared_mem_per_block_dynamic", "dyn smem"),
        ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes/inst")]
for k, n in keys:
    print(f"{n:20s} {d.get(k, '?')}")
st = {k.split("smsp__average_warp_latency_issue_stalled_")[1].split(".")[0]: g(k)
      for k in h if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")}
print("stalls/issue:", ", ".join(f"{k} {x:.2f}" for k, x in sorted(st.items(), key=lambda x: -x[1])[:9]))
