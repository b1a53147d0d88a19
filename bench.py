"""Benchmark: aligned curve pairs/sec (fp64, N=1024) on BASELINE config C1.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1]

One step = one pass of the hot path over one batch: 4096 pairs of raw curves
(n_in ~ U{300..3000}, non-uniform arc-length jitter, noise 1e-3) -> periodic
cubic spline resampling to N=1024 -> center/normalize -> FFT correlation ->
argmax -> rotation/energy/aligned curve, all in one sm_100a kernel launch.

* value: device-timed (CUDA events on the launching stream, max over ranks)
  whole-job pairs/s with inputs resident in HBM (inputs 216 MB > 126 MB L2).
* e2e: the same metric through the C-ABI host entry point
  (cva_preprocess_align_batch_host) from pinned host buffers, H2D of the raw
  curves and D2H of results + aligned curves inside the timed region.
* roofline: algorithmic HBM bytes per launch / mean launch time vs the measured
  copy bandwidth (MEASURED_PEAKS.json); fp64 side vs the FP64 peak measured here.
* cpu_baseline: the reference's own code (oracle/_ref, compiled in place against
  the FFTW/Eigen shims) on a bounded sample, all host threads.
Multi-GPU (torchrun): each rank aligns its own 4096-pair batch (weak scaling);
no data-path collective (pairs are independent).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aligned curve pairs/sec (fp64, N=1024)"
UNIT = "pairs/s"
WORKLOAD = "C1: 4096 pairs/GPU, raw n_in~U{300..3000} jittered arc length, noise 1e-3 -> N=1024, fp64"
E1_METRIC = "elastic distance pairs/sec (approach 2, fp64, N=256)"
E1_WORKLOAD = ("E1: distance_matrix(approach2) of 64 curves (raw n_in~U{300..3000}) preprocessed to N=256: "
               "4096 ordered pairs, max_iters 30, energy_tol 1e-6, max_slope 4")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=["c1", "c2", "c3", "c4", "e1"],
                    help="c1 is the headline (BASELINE metric); c2/c3/c4 are secondary workloads; "
                         "e1 is the elastic distance matrix (SURVEY.md 8(f))")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.ok = False
        self.samples, self.reasons = [], set()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_reference_run(pts, offs, pairs, N, seconds=12.0, threads=None, max_pairs=None):
    """Time the reference's own code (oracle/_ref) on a bounded sample; returns dict."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, Reference, reference_available

    kind = "reference" if reference_available() else "port"
    lib = Reference() if kind == "reference" else Oracle()
    threads = threads or (os.cpu_count() or 1)
    chunk = max(threads * 8, 64)
    done, t0 = 0, time.perf_counter()
    limit = max_pairs or pairs
    # whole passes over the batch until ~min_cpu_s of CPU work (threads x wall)
    # has been done, bounded by `seconds` of wall time
    min_cpu_s = 16.0
    while (time.perf_counter() - t0) < seconds:
        q = done % limit
        p1 = min(limit, q + chunk)
        sub = offs[2 * q:2 * p1 + 1] - offs[2 * q]
        lib.batch(pts[offs[2 * q]:offs[2 * p1]], sub, N, mode=0, threads=threads)
        done += p1 - q
        if done >= limit and (time.perf_counter() - t0) * threads >= min_cpu_s:
            break
    dt = time.perf_counter() - t0
    # single-thread figure on a short sample (T = 1 and T = all cores)
    t1_pairs, t1 = 0, time.perf_counter()
    while t1_pairs < limit and (time.perf_counter() - t1) < 4.0:
        p1 = min(limit, t1_pairs + 16)
        sub = offs[2 * t1_pairs:2 * p1 + 1] - offs[2 * t1_pairs]
        lib.batch(pts[offs[2 * t1_pairs]:offs[2 * p1]], sub, N, mode=0, threads=1)
        t1_pairs = p1
    dt1 = time.perf_counter() - t1
    return {"value": done / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "value_1_thread": t1_pairs / dt1, "cpu_model": cpu_model(),
            "sample": f"{done} C1 pairs ({done / limit:.1f} passes over the {limit}-pair batch) in {dt:.1f}s wall "
                      f"x {threads} threads = {dt * threads:.0f} CPU-s, "
                      + ("reference sources + FFTW/Eigen shims" if kind == "reference" else "C oracle port")}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return f"{os.cpu_count()} logical CPUs"


def algorithmic_bytes(offs, pairs, N):
    """Per launch: raw input read + offsets read + aligned curve write + result write."""
    raw = 16 * int(offs[2 * pairs] - offs[0])
    return raw + 8 * (2 * pairs + 1) + 16 * N * pairs + 48 * pairs


def run_reference_arm_e1(args):
    """The reference's elastic_distance_approach2 (oracle/_ref) on all host
    threads over a bounded sample of E1's ordered pairs per step."""
    from paper_2501_17779_b200 import synth

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference

    cfg = synth.CONFIGS["e1"]
    M, N = cfg["curves"], cfg["N"]
    pts, offs = synth.ragged_curves(args.seed, M)
    R = Reference()
    prep = np.stack([R.preprocess(pts[offs[c]:offs[c + 1]], N, True) for c in range(M)])
    threads = os.cpu_count() or 1
    sample = max(32, threads * 2)
    times, done = [], 0
    for it in range(args.warmup + args.steps):
        cells = (np.arange(sample) + it * sample) % (M * M)
        c1, c2 = prep[cells // M], prep[cells % M]
        t0 = time.perf_counter()
        R.elastic_approach2_batch(c1, c2, threads=threads)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
            done += sample
    total = sum(times)
    value = done / total
    line = {
        "impl": "reference", "metric": E1_METRIC, "value": value, "unit": UNIT, "n_gpus": dist_env()[1],
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C2 generator)",
        "config": {"workload": E1_WORKLOAD, "pairs_per_step": sample, "N": N},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{sample} E1 ordered pairs per step, reference elastic.cpp/srv.cpp sources"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.config == "e1":
        run_reference_arm_e1(args)
        return
    from paper_2501_17779_b200 import synth

    cfg = synth.CONFIGS["c1"]
    pairs, N = cfg["pairs"], cfg["N"]
    pts, offs, _, _ = synth.ragged_pairs(args.seed, pairs, N)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle, Reference, reference_available

    lib = Reference() if reference_available() else Oracle()
    threads = os.cpu_count() or 1
    sample = max(64, threads * 16)
    times, done = [], 0
    for i in range(args.warmup + args.steps):
        p0 = (i * sample) % pairs
        p1 = min(pairs, p0 + sample)
        sub = offs[2 * p0:2 * p1 + 1] - offs[2 * p0]
        t0 = time.perf_counter()
        lib.batch(pts[offs[2 * p0]:offs[2 * p1]], sub, N, mode=0, threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            done += p1 - p0
    total = sum(times)
    value = done / total
    kind = "reference" if reference_available() else "port"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C1 generator)",
        "config": {"workload": WORKLOAD, "pairs_per_step": sample, "N": N},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{sample} C1 pairs per step, reference sources + FFTW/Eigen shims"
                         if kind == "reference" else f"{sample} C1 pairs per step, C oracle port"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_secondary(args):
    """C2 (all pairs, N=512, FP64-bound) and C4 (SRV pairs, N=2048, HBM-bound):
    same JSON contract, device-timed, inputs resident."""
    import torch
    import torch.distributed as dist

    import paper_2501_17779_b200 as cva
    from paper_2501_17779_b200 import _native, synth

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _native.load()
    stream = torch.cuda.current_stream(dev)
    fp64 = ctypes_probe(lib)
    if args.config == "c2":
        cfg = synth.CONFIGS["c2"]
        M, N = cfg["curves"], cfg["N"]
        pts, offs = synth.ragged_curves(args.seed, M)
        dp, do = torch.from_numpy(pts).to(dev), torch.from_numpy(offs).to(dev)
        mx = int(np.diff(offs).max())
        r0, r1 = rank * M // world, (rank + 1) * M // world
        prep = torch.empty((M, N, 2), dtype=torch.float64, device=dev)
        e = torch.empty((r1 - r0, M), dtype=torch.float64, device=dev)
        k = torch.empty((r1 - r0, M), dtype=torch.int32, device=dev)
        th = torch.empty((r1 - r0, M), dtype=torch.float64, device=dev)

        if world > 1:  # the assembled matrices on every rank (one NCCL all-gather each)
            assert M % world == 0
            full = [torch.empty((M, M), dtype=x.dtype, device=dev) for x in (e, k, th)]

        def step():
            _native.check(lib.cva_preprocess_batch(dp.data_ptr(), do.data_ptr(), M, mx, N, 1, prep.data_ptr(), 0,
                                                   stream.cuda_stream))
            _native.check(lib.cva_allpairs(prep.data_ptr(), M, N, r0, r1, e.data_ptr(), k.data_ptr(), th.data_ptr(),
                                           stream.cuda_stream))
            if world > 1:
                for dst, src in zip(full, (e, k, th)):
                    dist.all_gather_into_tensor(dst, src)
        units = (r1 - r0) * M
        workload = (f"C2: all ordered pairs of {M} curves (raw n_in~U{{300..3000}}), N={N}, rows sharded, "
                    "matrices all-gathered (NCCL) inside the step when N > 1")
        l2 = "spectra (16.8 MB) L2-resident by design (reused by every cell); 4.2 M cells of output per step"
        flops_unit = 5 * N * math.log2(N)
        bound = "fp64"
    elif args.config == "c3":
        cfg = synth.CONFIGS["c3"]
        P, N = cfg["pairs"], cfg["N"]
        c1, c2, _, _ = synth.uniform_pairs(args.seed + 1000 * rank, P, N, cfg["modes"], cfg["amp"], cfg["amp_exp"],
                                           cfg["sigma"])
        d1, d2 = torch.from_numpy(c1).to(dev), torch.from_numpy(c2).to(dev)
        out = torch.empty((P, 48), dtype=torch.uint8, device=dev)
        al = torch.empty_like(d2)

        def step():
            _native.check(lib.cva_preprocess_align_uniform(d1.data_ptr(), d2.data_ptr(), P, N, out.data_ptr(),
                                                           al.data_ptr(), stream.cuda_stream))
        units = P
        workload = f"C3: {P} pairs/GPU, N={N}, center+normalize+align_fft+aligned curve (L2-chunked four-step FFT)"
        l2 = "inputs larger than L2 (2 x 268 MB curves + 268 MB aligned vs 126 MB)"
        bytes_unit = 16 * 2 * N + 16 * N + 48
        bound = "hbm"
    elif args.config == "e1":
        cfg = synth.CONFIGS["e1"]
        M, N = cfg["curves"], cfg["N"]
        pts, offs = synth.ragged_curves(args.seed, M)
        dp, do = torch.from_numpy(pts).to(dev), torch.from_numpy(offs).to(dev)
        mx = int(np.diff(offs).max())
        prep = torch.empty((M, N, 2), dtype=torch.float64, device=dev)
        d = torch.empty((M, M), dtype=torch.float64, device=dev)

        def step():
            _native.check(lib.cva_preprocess_batch(dp.data_ptr(), do.data_ptr(), M, mx, N, 1, prep.data_ptr(), 0,
                                                   stream.cuda_stream))
            _native.check(lib.cva_elastic_distance_matrix(prep.data_ptr(), M, N, 2, 30, 1e-6, 4, 512, d.data_ptr(),
                                                          stream.cuda_stream))
        units = M * M  # every rank computes the whole matrix (weak scaling: replicas)
        workload = E1_WORKLOAD
        l2 = "inputs L2-resident (64 curves); the DP is compute-bound"
        bound = "fp64ops"
    else:
        cfg = synth.CONFIGS["c4"]
        P, N = cfg["pairs"], cfg["N"]
        c1, c2, _, _, _ = synth.srv_pairs(args.seed + 1000 * rank, P, N)
        d1, d2 = torch.from_numpy(c1).to(dev), torch.from_numpy(c2).to(dev)
        out = torch.empty((P, 48), dtype=torch.uint8, device=dev)
        al = torch.empty_like(d2)

        def step():
            _native.check(lib.cva_srv_align_batch(d1.data_ptr(), d2.data_ptr(), P, N, out.data_ptr(), al.data_ptr(),
                                                  stream.cuda_stream))
        units = P
        workload = f"C4: {P} SRV pairs/GPU, N={N}, srv_transform+srv_center+align_fft+aligned q"
        l2 = "inputs larger than L2 (2 x 268 MB curves + 268 MB aligned vs 126 MB)"
        bytes_unit = 16 * 2 * N + 16 * N + 48
        bound = "hbm"
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    total_units = units * world
    value = total_units / (ms_step * 1e-3)
    launch_s = (ms / args.steps) * 1e-3
    if bound == "fp64ops":
        # FP64 thread ops (DADD + DMUL + DFMA) of the elastic kernel from its ncu
        # capture, per launch, against the FP64 op rate the probe measured
        # (dependent DFMA chains: TFLOP/s / 2 = T ops/s)
        prof = os.path.join(ROOT, "profiles", "r2h_e1_elastic_ncu_summary.json")
        ops = None
        if os.path.exists(prof):
            with open(prof) as f:
                ops = json.load(f).get("fp64_thread_ops_per_launch")
        ach = ops / launch_s / 1e12 if ops else None
        peak_ops = fp64 / 2 if fp64 else None
        roof = {"bound": "fp64", "achieved": ach, "peak": peak_ops, "unit": "T FP64 ops/s",
                "frac": ach / peak_ops if ach and peak_ops else None, "traffic": None,
                "peak_source": "measured here (cva_probe_fp64_tflops / 2)",
                "note": "DADD+DMUL+DFMA thread ops of the elastic kernel per launch (ncu, "
                        "profiles/r2h_e1_elastic_ncu_summary.json); the DP has no FFT-style flop model"}
    elif bound == "fp64":
        ach = units * flops_unit / launch_s / 1e12
        roof = {"bound": "fp64", "achieved": ach, "peak": fp64, "unit": "TFLOP/s", "frac": ach / fp64 if fp64 else None,
                "traffic": None, "peak_source": "measured here (cva_probe_fp64_tflops)",
                "note": "5 N log2 N flops per pair (one transform per cell; spectra amortised)"}
    else:
        hbm_peak, peak_kind = load_peaks()
        ach = units * bytes_unit / launch_s / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "traffic": None, "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"}
    if rank == 0:
        print(json.dumps({
            "metric": E1_METRIC if args.config == "e1" else f"aligned curve pairs/sec (fp64, {args.config})",
            "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if args.config == "c2" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, csrc/synth.cpp)",
            "config": {"workload": workload, "l2": l2}, "roofline": roof, "cpu_baseline": None, "e2e": None,
            "gpu_launches": args.steps * (2 if args.config in ("c2", "e1") else 1), "clocks": clk.summary()}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.config != "c1":
        run_secondary(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2501_17779_b200 as cva
    from paper_2501_17779_b200 import _native, synth

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _native.load()

    cfg = synth.CONFIGS["c1"]
    pairs, N = cfg["pairs"], cfg["N"]
    pts, offs, _, _ = synth.ragged_pairs(args.seed + 1000 * rank, pairs, N)
    max_n = int(np.diff(offs).max())
    dp = torch.from_numpy(pts).to(dev)
    do = torch.from_numpy(offs).to(dev)
    out = torch.empty((pairs, 48), dtype=torch.uint8, device=dev)
    al = torch.empty((pairs, N, 2), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        _native.check(lib.cva_preprocess_align_batch(dp.data_ptr(), do.data_ptr(), pairs, max_n, N, 1,
                                                     out.data_ptr(), al.data_ptr(), sptr))

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    res = cva.decode_results(out)
    assert (res["status"] == 0).all(), "kernel reported invalid pairs"

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = pairs * world / (ms_per_step * 1e-3)

    # ---- roofline (the single kernel of the step is the dominant kernel)
    hbm_peak, peak_kind = load_peaks()
    launch_s = (ms / args.steps) * 1e-3
    bytes_launch = algorithmic_bytes(offs, pairs, N)
    achieved_gbs = bytes_launch / launch_s / 1e9
    fp64 = ctypes_probe(lib)
    flops_launch = pairs * 3 * 5 * N * math.log2(N)
    traffic, ncu = None, {}
    prof = os.path.join(ROOT, "profiles", "ncu_c1_summary.json")
    if os.path.exists(prof):
        with open(prof) as f:
            ncu = json.load(f)
            traffic = ncu.get("dram_bytes_per_launch")
    roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved_gbs / hbm_peak, "traffic": traffic,
            "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
            "algorithmic_bytes_per_launch": bytes_launch,
            "fp64": {"achieved_tflops": flops_launch / launch_s / 1e12, "peak_tflops_measured": fp64,
                     "frac": (flops_launch / launch_s / 1e12) / fp64 if fp64 else None,
                     "flops_per_launch": flops_launch, "note": "15 N log2 N per pair (3 complex FFTs)"},
            # what actually binds (ncu capture of the same kernel, profiles/ncu_c1_summary.json)
            "binding": {"resource": "fp64 dependency latency / issue at 25 % occupancy (128 regs, 115 KB smem)",
                        "fp64_pipe_active_pct": ncu.get("sm__pipe_fp64_cycles_active_pct"),
                        "issue_slots_busy_pct": ncu.get("issue_slots_busy_pct"),
                        "l1tex_throughput_pct": ncu.get("l1tex_throughput_pct"),
                        # the kernel's own FP64 work (DADD+DMUL+DFMA thread ops,
                        # spline + FFTs) at the SMs' FP64 op rate: its compute
                        # floor, next to the HBM floor the fraction above uses
                        "fp64_thread_ops_per_pair": (round(ncu["fp64_thread_ops_per_launch"] / pairs)
                                                     if ncu.get("fp64_thread_ops_per_launch") else None),
                        "fp64_op_utilisation_pct": ncu.get("fp64_op_utilisation_pct"),
                        "ncu_round": ncu.get("round")}}

    # ---- end to end through the C-ABI host entry (pinned buffers)
    e2e = None
    if not args.no_e2e:
        hp = torch.from_numpy(pts).pin_memory()
        ho = torch.from_numpy(offs).pin_memory()
        hres = torch.empty((pairs, 48), dtype=torch.uint8).pin_memory()
        hal = torch.empty((pairs, N, 2), dtype=torch.float64).pin_memory()

        def e2e_step():
            _native.check(lib.cva_preprocess_align_batch_host(hp.data_ptr(), ho.data_ptr(), pairs, N, 1,
                                                              hres.data_ptr(), hal.data_ptr()))

        for _ in range(2):
            e2e_step()
        if world > 1:
            dist.barrier()
        k = max(3, min(args.steps, 20))
        t0 = time.perf_counter()
        for _ in range(k):
            e2e_step()
        dt = time.perf_counter() - t0
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
        e2e = {"value": pairs * world * k / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(pts.nbytes + offs.nbytes),
               "d2h_bytes_per_step": int(pairs * 48 + pairs * N * 16),
               "ms_per_step": 1e3 * dt / k, "timing": "host wall clock around synchronous C-ABI calls"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_run(pts, offs, pairs, N, seconds=12.0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded C1 generator, csrc/synth.cpp)",
            "config": {"workload": WORKLOAD, "pairs_per_gpu": pairs, "N": N, "n_in": [300, 3000],
                       "raw_points_per_gpu": int(offs[-1]),
                       "l2": "inputs larger than L2 (raw %.0f MB + aligned %.0f MB vs 126 MB)" % (
                           pts.nbytes / 1e6, pairs * N * 16 / 1e6)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ctypes_probe(lib):
    import ctypes

    v = ctypes.c_double(0.0)
    try:
        if lib.cva_probe_fp64_tflops(ctypes.addressof(v)) == 0:
            return v.value
    except Exception:
        pass
    return None


if __name__ == "__main__":
    main()
