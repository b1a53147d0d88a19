"""Per-kernel device time of one C3 step in the real pipeline (warm caches,
both chunk streams), via the CUDA profiler (CUPTI), beside the step's wall
time from CUDA events. Development tool: ncu's per-kernel numbers are cold
(caches flushed between replays) and serialised.

    python tools/c3_profile.py [--config c3|c4] [--steps 3]
"""
from __future__ import annotations

import argparse
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_17779_b200 import _native, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=["c3", "c4"])
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    P, N = cfg["pairs"], cfg["N"]
    if a.config == "c3":
        c1, c2, _, _ = synth.uniform_pairs(1, P, N, cfg["modes"], cfg["amp"], cfg["amp_exp"], cfg.get("sigma", 1e-3))
        fn = "cva_preprocess_align_uniform"
    else:
        c1, c2, _, _, _ = synth.srv_pairs(1, P, N)
        fn = "cva_srv_align_batch"
    lib = _native.load()
    d1, d2 = torch.from_numpy(c1).cuda(), torch.from_numpy(c2).cuda()
    out = torch.empty((P, 48), dtype=torch.uint8, device="cuda")
    al = torch.empty_like(d2)
    f = getattr(lib, fn)

    def step():
        _native.check(f(d1.data_ptr(), d2.data_ptr(), P, N, out.data_ptr(), al.data_ptr(),
                        torch.cuda.current_stream().cuda_stream))
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    wall = e0.elapsed_time(e1) / 10
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            step()
        torch.cuda.synchronize()
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name.split("(")[0][:70]
            tot[k] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            cnt[k] += 1
    print(f"{a.config}: step {wall * 1000:.1f} us (events, 10 steps)")
    s = 0.0
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        per = v / a.steps
        s += per
        print(f"  {k:72s} {per:9.1f} us/step  {cnt[k] / a.steps:6.1f} launches/step  {v / cnt[k]:7.2f} us each")
    print(f"  sum of kernel time {s:.1f} us/step (> step time = stream overlap)")


if __name__ == "__main__":
    main()
