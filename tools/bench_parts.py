"""Time the pieces of the C1 path separately (device-resident inputs, CUDA events).

    python tools/bench_parts.py [--pairs 4096] [--reps 20]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_17779_b200 import _native, synth  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--N", type=int, default=1024)
    a = ap.parse_args()
    lib = _native.load()
    pts, offs, _, _ = synth.ragged_pairs(1, a.pairs, a.N)
    dp = torch.from_numpy(pts).cuda()
    do = torch.from_numpy(offs).cuda()
    mx = int(np.diff(offs).max())
    s = torch.cuda.current_stream().cuda_stream
    N, P = a.N, a.pairs
    out = torch.empty((P, 48), dtype=torch.uint8, device="cuda")
    al = torch.empty((P, N, 2), dtype=torch.float64, device="cuda")
    prep = torch.empty((2 * P, N, 2), dtype=torch.float64, device="cuda")

    def fused():
        _native.check(lib.cva_preprocess_align_batch(dp.data_ptr(), do.data_ptr(), P, mx, N, 1, out.data_ptr(),
                                                     al.data_ptr(), s))

    def pre():
        _native.check(lib.cva_preprocess_batch(dp.data_ptr(), do.data_ptr(), 2 * P, mx, N, 1, prep.data_ptr(), 0, s))

    c1 = prep[0::2].contiguous()
    c2 = prep[1::2].contiguous()

    def align():
        _native.check(lib.cva_align_batch(c1.data_ptr(), c2.data_ptr(), P, N, out.data_ptr(), al.data_ptr(), s))

    def align_noal():
        _native.check(lib.cva_align_batch(c1.data_ptr(), c2.data_ptr(), P, N, out.data_ptr(), 0, s))

    for name, fn in (("fused resample+align", fused), ("preprocess 2P curves", pre),
                     ("align P pairs (+aligned)", align), ("align P pairs (no aligned)", align_noal)):
        ms = timeit(fn, a.reps)
        print(f"{name:28s} {ms * 1e3:9.1f} us   {P / (ms * 1e-3):12.0f} pairs/s")


if __name__ == "__main__":
    main()
