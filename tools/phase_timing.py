"""Per-phase cycle breakdown of the fused C1 kernel (needs `make prof`).

    python tools/phase_timing.py
Loads libcurvalign_cuda_prof.so (built with -DCVA_PHASE_TIMING) instead of the
shipped library and prints the mean cycles between consecutive stamps.
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_17779_b200 import _native, synth  # noqa: E402

_native.LIB_PATH = os.path.join(ROOT, "paper_2501_17779_b200", "libcurvalign_cuda_prof.so")
lib = _native.load()
lib.cva_debug_set_prof.argtypes = [ctypes.c_void_p]
P, N = 4096, 1024
pts, offs, _, _ = synth.ragged_pairs(1, P, N)
dp, do = torch.from_numpy(pts).cuda(), torch.from_numpy(offs).cuda()
mx = int(np.diff(offs).max())
out = torch.empty((P, 48), dtype=torch.uint8, device="cuda")
al = torch.empty((P, N, 2), dtype=torch.float64, device="cuda")
prof = torch.zeros((P, 64), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for it in range(3):
    assert lib.cva_debug_set_prof(prof.data_ptr() if it == 2 else 0) == 0
    _native.check(lib.cva_preprocess_align_batch(dp.data_ptr(), do.data_ptr(), P, mx, N, 1, out.data_ptr(),
                                                 al.data_ptr(), s))
torch.cuda.synchronize()
t = prof.cpu().numpy().astype(np.float64)
names = {0: "start", 1: "load A", 2: "A arc length", 3: "A phase1", 4: "A pcr", 7: "A p3 fwd (t0)",
         8: "A p3 bwd+eval (t0)", 5: "A p3 barrier wait", 6: "A len/centroid", 10: "load B", 11: "B arc length",
         12: "B phase1", 13: "B pcr", 16: "B p3 fwd (t0)", 17: "B p3 bwd+eval (t0)", 14: "B p3 barrier wait",
         15: "B len/centroid", 20: "2 FFTs", 21: "3rd FFT", 23: "argmax+aligned out"}
order = [0, 1, 2, 3, 4, 7, 8, 5, 6, 10, 11, 12, 13, 16, 17, 14, 15, 20, 21, 23]
tot = 0
for a, b in zip(order, order[1:]):
    d = t[:, b] - t[:, a]
    tot += d.mean()
    print(f"{names[b]:16s} {d.mean():9.0f} cycles (p50 {np.median(d):8.0f})")
print(f"{'total':16s} {tot:9.0f} cycles per CTA; n_in mean {np.diff(offs).mean():.0f}")
