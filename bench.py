"""Benchmark: aligned curve pairs/sec (fp64, N=1024) on BASELINE config C1.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4|e1] [--scaling weak|strong]

One step = one pass of the hot path over one batch: 4096 pairs of raw curves
(n_in ~ U{300..3000}, non-uniform arc-length jitter, noise 1e-3) -> periodic
cubic spline resampling to N=1024 -> center/normalize -> FFT correlation ->
argmax -> rotation/energy/aligned curve, all in one sm_100a kernel launch.

* --gpus N: one process per GPU. Without WORLD_SIZE in the environment and
  N > 1, bench.py relaunches itself under torch.distributed.run (127.0.0.1);
  under torchrun it checks WORLD_SIZE == N. Times are CUDA events on the
  launching stream, max over ranks; rank 0 prints the JSON line.
* C1 --scaling weak (default): every rank aligns its own 4096-pair batch;
  strong: the one 4096-pair batch split by pair ranges (shard_range). No
  data-path collective (pairs are independent).
* C2: rows of the 2048 x 2048 matrices sharded; each rank's rows computed in
  chunks and gathered to rank 0 with one NCCL gather of packed 20-byte cells
  per chunk, overlapping the next chunk (distributed.AllPairsGather).
* value: device-timed whole-job units/s with inputs resident in HBM.
* e2e: the same metric through the C-ABI host entry points (pinned host
  buffers, H2D of the inputs and D2H of the results inside the timed region).
* roofline: algorithmic bytes (or flops) per launch / mean launch time against
  MEASURED_PEAKS.json (HBM) or the FP64 rate measured on the box.
* cpu_baseline (rank 0, N = 1): the reference's own code (oracle/_ref, its
  sources compiled in place against the FFTW/Eigen shims) on a bounded sample,
  all host threads.
* --impl reference: the reference's CPU implementation of the configured
  workload (oracle/_ref), hermetic: the inputs are generated in a separate
  process, so no repo library is loaded into the timed process.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aligned curve pairs/sec (fp64, N=1024)"
UNIT = "pairs/s"
WORKLOAD = "C1: 4096 pairs/GPU, raw n_in~U{300..3000} jittered arc length, noise 1e-3 -> N=1024, fp64"
WORKLOAD_STRONG = "C1: one 4096-pair batch split over the GPUs, raw n_in~U{300..3000} -> N=1024, fp64"
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
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="C1 only: weak = 4096 pairs per GPU, strong = one 4096-pair batch split")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--selftest", action="store_true",
                    help="CPU-only launcher / collective check (gloo, stand-in compute; tests/)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int | None:
    """--gpus N > 1 without a torchrun environment: run N ranks of this script
    under torch.distributed.run and return its exit code (rank 0's JSON line
    goes to our stdout). Under torchrun: None (after checking WORLD_SIZE)."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus and not (args.gpus == 1 and world == 1):
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
            raise SystemExit(2)
        return None
    if args.gpus <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return f"{os.cpu_count()} logical CPUs"


SHIM_NOTE = ("reference sources compiled in place against builder-written FFTW3/Eigen shims "
             "(oracle/shim: plan-cached twiddles, r2c/c2r via a half-length complex transform; "
             "real FFTW is not in the image)")


# --------------------------------------------------------------------------- workloads

def gen_inputs(config: str, seed: int, rank: int = 0):
    """The seeded synthetic inputs of a config (csrc/synth.cpp via synth.py)."""
    from paper_2501_17779_b200 import synth

    cfg = synth.CONFIGS[config]
    s = seed + 1000 * rank
    if config == "c1":
        pts, offs, _, _ = synth.ragged_pairs(s, cfg["pairs"], cfg["N"])
        return {"pts": pts, "offs": offs}
    if config in ("c2", "e1"):
        pts, offs = synth.ragged_curves(seed, cfg["curves"])
        return {"pts": pts, "offs": offs}
    if config == "c3":
        c1, c2, _, _ = synth.uniform_pairs(s, cfg["pairs"], cfg["N"], cfg["modes"], cfg["amp"], cfg["amp_exp"],
                                           cfg["sigma"])
        return {"c1": c1, "c2": c2}
    c1, c2, _, _, _ = synth.srv_pairs(s, cfg["pairs"], cfg["N"])
    return {"c1": c1, "c2": c2}


def gen_inputs_isolated(config: str, seed: int) -> dict:
    """gen_inputs in a child process (the reference arm stays free of repo
    libraries); arrays come back through an .npz file."""
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "inputs.npz")
        code = ("import sys, numpy as np; sys.path.insert(0, %r); import bench; "
                "np.savez(%r, **bench.gen_inputs(%r, %d))" % (ROOT, path, config, seed))
        subprocess.run([sys.executable, "-c", code], check=True)
        with np.load(path) as z:
            return {k: z[k] for k in z.files}


def pairs_ragged(c1, c2):
    """Interleave uniform pairs as the ragged layout of ref_batch (curve 2p, 2p+1)."""
    P, N = c1.shape[0], c1.shape[1]
    pts = np.empty((P, 2, N, 2))
    pts[:, 0], pts[:, 1] = c1, c2
    return pts.reshape(-1, 2), np.arange(2 * P + 1, dtype=np.int64) * N


class RefRunner:
    """The reference's own implementation (oracle/_ref) on host threads, one
    bounded sample of a config's workload per call. Units per sample are
    returned with the call so rates are units / seconds."""

    def __init__(self, config, inputs, threads=None):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from paper_2501_17779_b200 import synth
        from pyoracle import Oracle, Reference, reference_available

        self.kind = "reference" if reference_available() else "port"
        self.lib = Reference() if self.kind == "reference" else Oracle()
        self.threads = threads or (os.cpu_count() or 1)
        self.config, self.inp = config, inputs
        self.cfg = synth.CONFIGS[config]
        self.i = 0
        t = self.threads
        if config == "c1":
            self.P, self.N = self.cfg["pairs"], self.cfg["N"]
            self.sample = max(64, 16 * t)
            self.what = f"{self.sample} C1 pairs per call (preprocess both + align_fft)"
        elif config == "c2":
            # the reference preprocesses every curve once, then aligns the cells
            M, N = self.cfg["curves"], self.cfg["N"]
            pts, offs = inputs["pts"], inputs["offs"]
            t0 = time.perf_counter()
            self.prep = np.stack([self.lib.preprocess(pts[offs[c]:offs[c + 1]], N, True) for c in range(M)])
            self.prep_s = time.perf_counter() - t0  # single thread
            self.M = M
            self.rows = max(1, (2 * t) // 1)
            self.sample = self.rows * M
            self.what = (f"{self.rows} full rows ({self.sample} cells) per call + the per-cell share of "
                         f"preprocessing all {M} curves ({self.prep_s:.2f} s, one thread)")
        elif config == "c3":
            self.sample = max(4, t // 2)
            self.what = f"{self.sample} C3 pairs per call (center+normalize+align_fft, N=65536)"
        elif config == "c4":
            self.sample = max(64, 16 * t)
            self.what = f"{self.sample} C4 pairs per call (srv_transform+srv_center+align_fft, N=2048)"
        else:
            M, N = self.cfg["curves"], self.cfg["N"]
            pts, offs = inputs["pts"], inputs["offs"]
            self.prep = np.stack([self.lib.preprocess(pts[offs[c]:offs[c + 1]], N, True) for c in range(M)])
            self.M = M
            self.sample = max(32, 2 * t)
            self.what = f"{self.sample} E1 ordered pairs per call (elastic_distance_approach2)"

    def call(self, threads=None) -> tuple[int, float]:
        t = threads or self.threads
        i, self.i = self.i, self.i + 1
        if self.config == "c1":
            pts, offs = self.inp["pts"], self.inp["offs"]
            p0 = (i * self.sample) % self.P
            p1 = min(self.P, p0 + self.sample)
            sub = offs[2 * p0:2 * p1 + 1] - offs[2 * p0]
            t0 = time.perf_counter()
            self.lib.batch(pts[offs[2 * p0]:offs[2 * p1]], sub, self.N, mode=0, threads=t)
            return p1 - p0, time.perf_counter() - t0
        if self.config == "c2":
            r0 = (i * self.rows) % self.M
            r1 = min(self.M, r0 + self.rows)
            t0 = time.perf_counter()
            self.lib.allpairs(self.prep, r0, r1, threads=t)
            dt = time.perf_counter() - t0
            cells = (r1 - r0) * self.M
            return cells, dt + self.prep_s / t * cells / (self.M * self.M)
        if self.config in ("c3", "c4"):
            P, N = self.inp["c1"].shape[0], self.inp["c1"].shape[1]
            p0 = (i * self.sample) % P
            p1 = min(P, p0 + self.sample)
            pts, offs = pairs_ragged(self.inp["c1"][p0:p1], self.inp["c2"][p0:p1])
            t0 = time.perf_counter()
            if self.config == "c3":
                self.lib.batch(pts, offs, N, mode=0, resample=False, threads=t)
            else:
                self.lib.batch(pts, offs, N, mode=2, threads=t)
            return p1 - p0, time.perf_counter() - t0
        cells = (np.arange(self.sample) + i * self.sample) % (self.M * self.M)
        c1, c2 = self.prep[cells // self.M], self.prep[cells % self.M]
        t0 = time.perf_counter()
        self.lib.elastic_approach2_batch(c1, c2, threads=t)
        return self.sample, time.perf_counter() - t0


def cpu_baseline(config, inputs, seconds=12.0) -> dict:
    """The reference on all host threads over ~min(seconds) of samples, plus a
    single-thread figure (T = 1 and T = all cores)."""
    rr = RefRunner(config, inputs)
    done, dt = 0, 0.0
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < seconds:
        u, s = rr.call()
        done, dt = done + u, dt + s
        if dt * rr.threads >= 16.0:
            break
    u1, s1 = 0, 0.0
    while s1 < 3.0:
        u, s = rr.call(threads=1)
        u1, s1 = u1 + u, s1 + s
        if config in ("c3",):
            break
    return {"value": done / dt, "unit": UNIT, "cores": rr.threads, "kind": rr.kind, "value_1_thread": u1 / s1,
            "cpu_model": cpu_model(),
            "sample": f"{done} units in {dt:.1f} s x {rr.threads} threads; {rr.what}; {SHIM_NOTE}"}


# --------------------------------------------------------------------------- reference arm

METRICS = {"c1": METRIC, "c2": "aligned curve pairs/sec (fp64, c2)", "c3": "aligned curve pairs/sec (fp64, c3)",
           "c4": "aligned curve pairs/sec (fp64, c4)", "e1": E1_METRIC}


def workload_of(config, scaling="weak"):
    from_cfg = {
        "c1": WORKLOAD if scaling == "weak" else WORKLOAD_STRONG,
        "c2": "C2: all ordered pairs of 2048 curves (raw n_in~U{300..3000}), N=512, rows sharded, "
              "row chunks gathered to rank 0 (NCCL) when N > 1",
        "c3": "C3: 256 pairs/GPU, N=65536, center+normalize+align_fft+aligned curve",
        "c4": "C4: 8192 SRV pairs/GPU, N=2048, srv_transform+srv_center+align_fft+aligned q",
        "e1": E1_WORKLOAD,
    }
    return from_cfg[config]


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    inputs = gen_inputs_isolated(args.config, args.seed)
    rr = RefRunner(args.config, inputs)
    times, done = [], 0
    for i in range(args.warmup + args.steps):
        u, dt = rr.call()
        if i >= args.warmup:
            times.append(dt)
            done += u
    total = sum(times)
    value = done / total
    line = {
        "impl": "reference", "metric": METRICS[args.config], "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, generated in a separate process)",
        "config": {"workload": workload_of(args.config, args.scaling), "units_per_step": rr.sample,
                   "threads": rr.threads, "cpu_model": cpu_model()},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": rr.threads, "kind": rr.kind,
                         "sample": f"{rr.what}; {SHIM_NOTE}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_libs_loaded": repo_libs_loaded(),
    }
    print(json.dumps(line), flush=True)


def repo_libs_loaded():
    """Shared objects of this repo mapped into the process (the reference arm:
    only oracle/_ref, the reference's own sources)."""
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                path = line.split()[-1] if line.strip() else ""
                if path.endswith(".so") and os.path.realpath(path).startswith(os.path.realpath(ROOT)):
                    libs.add(os.path.relpath(os.path.realpath(path), os.path.realpath(ROOT)))
    except OSError:
        pass
    return sorted(libs)


# --------------------------------------------------------------------------- GPU arm

def ctypes_probe(lib):
    import ctypes

    v = ctypes.c_double(0.0)
    try:
        if lib.cva_probe_fp64_tflops(ctypes.addressof(v)) == 0:
            return v.value
    except Exception:
        pass
    return None


def algorithmic_bytes_c1(offs, p0, p1, N):
    """Per launch: raw input read + offsets read + aligned curve write + result write."""
    pairs = p1 - p0
    raw = 16 * int(offs[2 * p1] - offs[2 * p0])
    return raw + 8 * (2 * pairs + 1) + 16 * N * pairs + 48 * pairs


def ncu_summary(name):
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def time_steps(step, steps, warmup, stream, local, world, dist):
    """Warm-up, then `steps` steps between CUDA events on `stream`, barrier +
    synchronize on both sides; returns (max-over-ranks ms for all steps,
    this rank's ms, clock summary)."""
    import torch

    for _ in range(max(3, warmup)):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=torch.device("cuda", local))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), ms, clk.summary()


def count_kernels(step):
    """Kernels of this library (namespace cva) that one step launches, counted
    by the CUDA profiler outside the timed region (NCCL / torch kernels are
    not ours and not counted)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    try:
        step()  # first-call setup (twiddle tables, workspaces) is not a step
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
            step()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events()
                 if e.device_type == torch.autograd.DeviceType.CUDA and "cva::" in e.name]
        count_kernels.names = sorted(set(n.split("(")[0] for n in names))
        return len(names)
    except Exception:
        return None


def graph_of(step):
    """One step captured as a CUDA graph; returns its replay on the current stream."""
    import torch

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()  # warm on the capture stream (first-call setup is not capturable)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    torch.cuda.synchronize()
    graph_of.keep = g
    return g.replay


def wall_max(seconds, world, dist, local):
    import torch

    t = torch.tensor([seconds], dtype=torch.float64, device=torch.device("cuda", local))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2501_17779_b200 as cva
    from paper_2501_17779_b200 import _native, synth
    from paper_2501_17779_b200.distributed import AllPairsGather, shard_range

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _native.load()
    stream = torch.cuda.current_stream(dev)

    def cs():  # the current stream at call time (a graph capture switches it)
        return torch.cuda.current_stream(dev).cuda_stream
    fp64 = ctypes_probe(lib)
    cfg = synth.CONFIGS[args.config]
    strong = args.config == "c1" and args.scaling == "strong"
    inputs = gen_inputs(args.config, args.seed, 0 if (strong or args.config in ("c2", "e1")) else rank)
    launches_per_step = 1
    e2e_fn, e2e_bytes = None, (0, 0)

    if args.config == "c1":
        P, N = cfg["pairs"], cfg["N"]
        pts, offs = inputs["pts"], inputs["offs"]
        p0, p1 = shard_range(P, rank, world) if strong else (0, P)
        lp = offs[2 * p0:2 * p1 + 1] - offs[2 * p0]
        lpts = np.ascontiguousarray(pts[offs[2 * p0]:offs[2 * p1]])
        pairs = p1 - p0
        max_n = int(np.diff(lp).max())
        dp, do = torch.from_numpy(lpts).to(dev), torch.from_numpy(lp).to(dev)
        out = torch.empty((pairs, 48), dtype=torch.uint8, device=dev)
        al = torch.empty((pairs, N, 2), dtype=torch.float64, device=dev)

        def step():
            _native.check(lib.cva_preprocess_align_batch(dp.data_ptr(), do.data_ptr(), pairs, max_n, N, 1,
                                                         out.data_ptr(), al.data_ptr(), cs()))
        units = pairs
        bytes_launch = algorithmic_bytes_c1(offs, p0, p1, N)
        flops_launch = pairs * 3 * 5 * N * math.log2(N)
        bound = "hbm"

        hp, ho = torch.from_numpy(lpts).pin_memory(), torch.from_numpy(lp).pin_memory()
        hres = torch.empty((pairs, 48), dtype=torch.uint8).pin_memory()
        hal = torch.empty((pairs, N, 2), dtype=torch.float64).pin_memory()

        def e2e_fn():
            _native.check(lib.cva_preprocess_align_batch_host(hp.data_ptr(), ho.data_ptr(), pairs, N, 1,
                                                              hres.data_ptr(), hal.data_ptr()))
        e2e_bytes = (int(lpts.nbytes + lp.nbytes), int(pairs * 48 + pairs * N * 16))
    elif args.config == "c2":
        M, N = cfg["curves"], cfg["N"]
        pts, offs = inputs["pts"], inputs["offs"]
        dp, do = torch.from_numpy(pts).to(dev), torch.from_numpy(offs).to(dev)
        mx = int(np.diff(offs).max())
        prep = torch.empty((M, N, 2), dtype=torch.float64, device=dev)
        r0, r1 = shard_range(M, rank, world)

        def prep_step():
            _native.check(lib.cva_preprocess_batch(dp.data_ptr(), do.data_ptr(), M, mx, N, 1, prep.data_ptr(), 0,
                                                   cs()))
        if world > 1:
            def fill(rb, re, e, k, th):
                _native.check(lib.cva_allpairs(prep.data_ptr(), M, N, rb, re, e.data_ptr(), k.data_ptr(),
                                               th.data_ptr(), cs()))
            gat = AllPairsGather(M, fill, chunks=4, dst=0)

            def step():
                prep_step()
                gat.run()
            launches_per_step = 1 + 4
        else:
            e = torch.empty((M, M), dtype=torch.float64, device=dev)
            k = torch.empty((M, M), dtype=torch.int32, device=dev)
            th = torch.empty((M, M), dtype=torch.float64, device=dev)

            def step():
                prep_step()
                _native.check(lib.cva_allpairs(prep.data_ptr(), M, N, 0, M, e.data_ptr(), k.data_ptr(),
                                               th.data_ptr(), cs()))
            launches_per_step = 2
        units = (r1 - r0) * M
        flops_unit = 5 * N * math.log2(N)
        bound = "fp64"

        hp, ho = torch.from_numpy(pts).pin_memory(), torch.from_numpy(offs).pin_memory()
        hprep = torch.empty((M, N, 2), dtype=torch.float64).pin_memory()
        he = torch.empty((r1 - r0, M), dtype=torch.float64).pin_memory()
        hk = torch.empty((r1 - r0, M), dtype=torch.int32).pin_memory()
        hth = torch.empty((r1 - r0, M), dtype=torch.float64).pin_memory()

        def e2e_fn():  # the user's flow: preprocess the curves, then this rank's rows of the matrices
            _native.check(lib.cva_preprocess_batch_host(hp.data_ptr(), ho.data_ptr(), M, N, 1, hprep.data_ptr(), 0))
            _native.check(lib.cva_allpairs_host(hprep.data_ptr(), M, N, r0, r1, he.data_ptr(), hk.data_ptr(),
                                                hth.data_ptr()))
        e2e_bytes = (int(pts.nbytes + offs.nbytes + M * N * 16), int(M * N * 16 + (r1 - r0) * M * 20))
    elif args.config in ("c3", "c4"):
        P, N = cfg["pairs"], cfg["N"]
        c1, c2 = inputs["c1"], inputs["c2"]
        d1, d2 = torch.from_numpy(c1).to(dev), torch.from_numpy(c2).to(dev)
        out = torch.empty((P, 48), dtype=torch.uint8, device=dev)
        al = torch.empty_like(d2)
        dev_fn = lib.cva_preprocess_align_uniform if args.config == "c3" else lib.cva_srv_align_batch
        host_fn = lib.cva_preprocess_align_uniform_host if args.config == "c3" else lib.cva_srv_align_batch_host

        def step():
            _native.check(dev_fn(d1.data_ptr(), d2.data_ptr(), P, N, out.data_ptr(), al.data_ptr(), cs()))
        units = P
        bytes_launch = P * (16 * 2 * N + 16 * N + 48)
        bound = "hbm"
        hc1, hc2 = torch.from_numpy(c1).pin_memory(), torch.from_numpy(c2).pin_memory()
        hres = torch.empty((P, 48), dtype=torch.uint8).pin_memory()
        hal = torch.empty((P, N, 2), dtype=torch.float64).pin_memory()

        def e2e_fn():
            _native.check(host_fn(hc1.data_ptr(), hc2.data_ptr(), P, N, hres.data_ptr(), hal.data_ptr()))
        e2e_bytes = (int(c1.nbytes + c2.nbytes), int(P * 48 + P * N * 16))
    else:  # e1
        M, N = cfg["curves"], cfg["N"]
        pts, offs = inputs["pts"], inputs["offs"]
        dp, do = torch.from_numpy(pts).to(dev), torch.from_numpy(offs).to(dev)
        mx = int(np.diff(offs).max())
        prep = torch.empty((M, N, 2), dtype=torch.float64, device=dev)
        d = torch.empty((M, M), dtype=torch.float64, device=dev)

        def step():
            _native.check(lib.cva_preprocess_batch(dp.data_ptr(), do.data_ptr(), M, mx, N, 1, prep.data_ptr(), 0,
                                                   cs()))
            _native.check(lib.cva_elastic_distance_matrix(prep.data_ptr(), M, N, 2, 30, 1e-6, 4, 512, d.data_ptr(),
                                                          cs()))
        units = M * M  # every rank computes the whole matrix (replicas)
        bound = "fp64ops"
        launches_per_step = 2
        hp, ho = torch.from_numpy(pts).pin_memory(), torch.from_numpy(offs).pin_memory()
        hprep = torch.empty((M, N, 2), dtype=torch.float64).pin_memory()
        hd = torch.empty((M, M), dtype=torch.float64).pin_memory()

        def e2e_fn():
            _native.check(lib.cva_preprocess_batch_host(hp.data_ptr(), ho.data_ptr(), M, N, 1, hprep.data_ptr(), 0))
            _native.check(lib.cva_elastic_distance_matrix_host(hprep.data_ptr(), M, N, 2, 30, 1e-6, 4, 512,
                                                               hd.data_ptr()))
        e2e_bytes = (int(pts.nbytes + offs.nbytes + M * N * 16), int(M * N * 16 + M * M * 8))

    launches_per_step = count_kernels(step) or launches_per_step

    # multi-kernel steps replay as one CUDA graph (same kernels, no launch gaps);
    # the NCCL gathers of C2 at N > 1 stay eager
    use_graph = args.config in ("c2", "c3", "e1") and world == 1
    timed = graph_of(step) if use_graph else step
    ms_max, ms_own, clocks = time_steps(timed, args.steps, args.warmup, stream, local, world, dist)
    if args.config == "c1":
        res = cva.decode_results(out)
        assert (res["status"] == 0).all(), "kernel reported invalid pairs"
    ms_step = ms_max / args.steps
    total_units = units * world if args.config != "e1" else units * world
    value = total_units / (ms_step * 1e-3)
    launch_s = (ms_own / args.steps) * 1e-3

    if bound == "hbm":
        hbm_peak, peak_kind = load_peaks()
        ach = bytes_launch / launch_s / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "traffic": None, "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "algorithmic_bytes_per_launch": bytes_launch}
        if args.config == "c1":
            ncu = ncu_summary("ncu_c1_summary.json")
            roof["traffic"] = ncu.get("dram_bytes_per_launch") if world == 1 and not strong else None
            roof["fp64"] = {"achieved_tflops": flops_launch / launch_s / 1e12, "peak_tflops_measured": fp64,
                            "frac": (flops_launch / launch_s / 1e12) / fp64 if fp64 else None,
                            "flops_per_launch": flops_launch, "note": "15 N log2 N per pair (3 complex FFTs)"}
            roof["binding"] = {
                "resource": "FP64 issue / dependency latency (see DESIGN.md 4.1)",
                "fp64_pipe_active_pct": ncu.get("sm__pipe_fp64_cycles_active_pct"),
                "issue_slots_busy_pct": ncu.get("issue_slots_busy_pct"),
                "fp64_thread_ops_per_pair": (round(ncu["fp64_thread_ops_per_launch"] / 4096)
                                             if ncu.get("fp64_thread_ops_per_launch") else None),
                "fp64_op_utilisation_pct": ncu.get("fp64_op_utilisation_pct"),
                "ncu_round": ncu.get("round"), "ncu_commit": ncu.get("commit")}
        else:
            ncu = ncu_summary(f"ncu_{args.config}_summary.json")
            roof["traffic"] = ncu.get("dram_bytes_per_launch")
            roof["note"] = "algorithmic bytes: 2 input curves + aligned curve + 48 B result per pair"
    elif bound == "fp64":
        ach = units * flops_unit / launch_s / 1e12
        ncu = ncu_summary("ncu_c2_summary.json")
        roof = {"bound": "fp64", "achieved": ach, "peak": fp64, "unit": "TFLOP/s", "frac": ach / fp64 if fp64 else None,
                "traffic": ncu.get("dram_bytes_per_launch"), "peak_source": "measured here (cva_probe_fp64_tflops)",
                "note": "5 N log2 N flops per cell (one transform per cell; spectra amortised); the step also "
                        "preprocesses all curves" + (" and gathers the rows to rank 0" if world > 1 else "")}
    else:
        prof = ncu_summary("r2h_e1_elastic_ncu_summary.json")
        ops = prof.get("fp64_thread_ops_per_launch")
        ach = ops / launch_s / 1e12 if ops else None
        peak_ops = fp64 / 2 if fp64 else None
        roof = {"bound": "fp64", "achieved": ach, "peak": peak_ops, "unit": "T FP64 ops/s",
                "frac": ach / peak_ops if ach and peak_ops else None, "traffic": None,
                "peak_source": "measured here (cva_probe_fp64_tflops / 2)",
                "note": "DADD+DMUL+DFMA thread ops of the elastic kernel per launch (ncu, "
                        "profiles/r2h_e1_elastic_ncu_summary.json); the DP has no FFT-style flop model"}

    # ---- end to end through the C-ABI host entry points (pinned buffers)
    e2e = None
    if not args.no_e2e and e2e_fn is not None:
        for _ in range(2):
            e2e_fn()
        if world > 1:
            dist.barrier()
        k = max(3, min(args.steps, 20 if args.config != "c3" else 5))
        t0 = time.perf_counter()
        for _ in range(k):
            e2e_fn()
        dt = wall_max(time.perf_counter() - t0, world, dist, local)
        e2e = {"value": units * world * k / dt, "unit": UNIT, "h2d_bytes_per_step": e2e_bytes[0],
               "d2h_bytes_per_step": e2e_bytes[1], "ms_per_step": 1e3 * dt / k,
               "timing": "host wall clock around synchronous C-ABI *_host calls, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, inputs if args.config != "c1" else {"pts": pts, "offs": offs})

    if rank == 0:
        line = {
            "metric": METRICS[args.config], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if (strong or args.config == "c2") else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, csrc/synth.cpp)",
            "config": {"workload": workload_of(args.config, args.scaling), "units_per_gpu": units,
                       "l2": ("inputs larger than L2" if args.config in ("c1", "c3", "c4")
                              else "spectra / curves L2-resident by design")},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks, "kernels": getattr(count_kernels, "names", None), "cuda_graph": use_graph,
        }
        if args.config == "c1":
            line["config"].update({"pairs_per_gpu": units, "N": cfg["N"], "n_in": [300, 3000],
                                   "raw_points_per_gpu": int(offs[2 * p1] - offs[2 * p0])})
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------------------- CPU self-test

def run_selftest(args):
    """No GPU: the launcher, rank/world plumbing, the max-over-ranks timing and
    the C2 chunked gather to rank 0 over gloo, with a CPU stand-in for the
    kernels (tests/test_bench_launcher.py)."""
    import torch
    import torch.distributed as dist

    from paper_2501_17779_b200.distributed import AllPairsGather, shard_range

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    M = 37

    def fill(rb, re, e, k, th):  # cell (i, j) -> deterministic values
        i = torch.arange(rb, re, dtype=torch.float64)[:, None]
        j = torch.arange(M, dtype=torch.float64)[None, :]
        e.copy_(i * M + j)
        k.copy_((i * 3 + j).to(torch.int32))
        th.copy_(-(i * M + j))

    ok = True
    t0 = time.perf_counter()
    for _ in range(args.warmup + args.steps):
        if world > 1:
            g = AllPairsGather(M, fill, chunks=3, dst=0)
            g.run()
            got = g.assemble()
        else:
            e = torch.empty((M, M), dtype=torch.float64)
            k = torch.empty((M, M), dtype=torch.int32)
            th = torch.empty((M, M), dtype=torch.float64)
            fill(0, M, e, k, th)
            got = (e, k, th)
        if rank == 0:
            i = torch.arange(M, dtype=torch.float64)[:, None]
            j = torch.arange(M, dtype=torch.float64)[None, :]
            ok &= bool(torch.equal(got[0], i * M + j) and torch.equal(got[1], (i * 3 + j).to(torch.int32))
                       and torch.equal(got[2], -(i * M + j)))
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": "selftest", "value": M * M * (args.warmup + args.steps) / float(t.item()),
                          "unit": "cells/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "selftest_ok": ok, "shares": [shard_range(M, r, world) for r in range(world)]}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rc = relaunch(args)
    if rc is not None:
        raise SystemExit(rc)
    if args.selftest:
        run_selftest(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
