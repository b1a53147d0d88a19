"""Time the elastic kernels' parts: one DP per pair vs the full approach-2 search.

    python tools/elastic_parts.py [--pairs 4096] [--n 256]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_17779_b200 as cva  # noqa: E402
from paper_2501_17779_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", type=int, default=4096)
ap.add_argument("--n", type=int, default=256)
a = ap.parse_args()
pts, offs = synth.ragged_curves(7, 64)
prep, _ = cva.preprocess_batch(pts, offs, a.n)
idx = np.arange(a.pairs)
c1 = torch.from_numpy(prep[idx // 64 % 64]).cuda()
c2 = torch.from_numpy(prep[idx % 64]).cuda()
q1 = torch.from_numpy(np.stack([cva.api._f64c(p) for p in prep])).cuda()


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


# SRV inputs for the DP: srv of the curves (reference formula) via the C4 helper path
from paper_2501_17779_b200 import _native  # noqa: E402

lib = _native.load()
ms_dp, _ = timeit(lambda: cva.dp_reparam_batch(c1, c2))  # DP on the curves themselves (same work shape)
ms_a2, r = timeit(lambda: cva.elastic_approach2_batch(c1, c2))
it = r["iterations"].cpu().numpy()
print(f"n={a.n} pairs={a.pairs}: one DP per pair {ms_dp:.2f} ms; approach 2 {ms_a2:.2f} ms "
      f"(mean iterations {it.mean():.2f}, DPs {it.sum()}) -> {ms_a2 / max(it.sum(), 1) * 1e3:.2f} us/DP-equivalent")
ms_m, _ = timeit(lambda: cva.elastic_distance_matrix(torch.from_numpy(prep).cuda()))
print(f"matrix mode (64 curves): {ms_m:.2f} ms")
pts1, offs1 = synth.ragged_curves(1, 64)
prep1, _ = cva.preprocess_batch(pts1, offs1, a.n)
ms_m1, r1 = timeit(lambda: cva.elastic_distance_matrix(torch.from_numpy(prep1).cuda()))
i1 = np.arange(4096)
r1b = cva.elastic_approach2_batch(prep1[i1 // 64], prep1[i1 % 64])
print(f"matrix mode seed 1: {ms_m1:.2f} ms; mean iterations {r1b['iterations'].mean():.2f}")
