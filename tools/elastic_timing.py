"""Time the GPU elastic distance matrix (approach 2) against the reference's
CPU code on a bounded sample.

    python tools/elastic_timing.py [--count 64] [--n 256] [--cpu-pairs 64]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2501_17779_b200 as cva  # noqa: E402
from paper_2501_17779_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--count", type=int, default=64)
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--cpu-pairs", type=int, default=64)
a = ap.parse_args()

pts, offs = synth.ragged_curves(7, a.count)
prep, st = cva.preprocess_batch(pts, offs, a.n)
assert (st == 0).all()
dc = torch.from_numpy(prep).cuda()
cva.elastic_distance_matrix(dc[:4])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
d = cva.elastic_distance_matrix(dc)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
pairs = a.count * a.count
print(f"GPU: {pairs} pairs n={a.n} in {ms:.1f} ms -> {pairs / ms * 1e3:.0f} pairs/s")
from pyoracle import Reference  # noqa: E402

R = Reference()
k = int(np.sqrt(a.cpu_pairs))
i, j = np.meshgrid(np.arange(k), np.arange(k), indexing="ij")
c1, c2 = prep[i.ravel()], prep[j.ravel()]
th = os.cpu_count() or 1
t = time.perf_counter()
r = R.elastic_approach2_batch(c1, c2, threads=th)
dt = time.perf_counter() - t
print(f"CPU reference: {k * k} pairs, {th} threads in {dt:.2f} s -> {k * k / dt:.1f} pairs/s")
g = d.cpu().numpy()[:k, :k].ravel()
rel = np.abs(g - r["distance"]) / np.maximum(np.abs(r["distance"]), 1e-300)
print(f"max rel diff vs reference on the sample: {np.nanmax(rel[r['distance'] > 0]):.3e}; "
      f"iterations equal: {(cva.elastic_approach2_batch(c1, c2)['iterations'] == r['iterations']).mean():.3f}")
