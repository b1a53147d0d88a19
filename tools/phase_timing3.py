"""Per-phase cycle breakdown of the v3 fused C1 kernel (needs `make prof`).

    python tools/phase_timing3.py
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
names = {0: "start", 1: "load A", 2: "A sweep+scan", 3: "A xchg", 4: "A pcr", 5: "A p3+map", 6: "A eval+sum",
         10: "load B", 11: "B sweep+scan", 12: "B xchg", 13: "B pcr", 14: "B p3+map", 15: "B eval+sum",
         20: "2 FFTs", 21: "3rd FFT", 23: "argmax+aligned out"}
order = [0, 1, 2, 3, 4, 5, 6, 10, 11, 12, 13, 14, 15, 20, 21, 23]
tot = 0
for a, b in zip(order, order[1:]):
    d = t[:, b] - t[:, a]
    tot += d.mean()
    print(f"{names[b]:20s} {d.mean():9.0f} cycles (p50 {np.median(d):8.0f})")
print(f"{'total':20s} {tot:9.0f} cycles per CTA; n_in mean {np.diff(offs).mean():.0f}")

sub = [(1, 34, "A merged sweep"), (34, 2, "A scan+knots"), (2, 3, "A xchg barrier"), (4, 37, "A p3 fwd"),
       (37, 38, "A p3 bwd"),
       (38, 5, "A p3 barrier"), (5, 35, "A map scan"), (35, 36, "A eval"), (36, 6, "A block sum")]
print("-- curve A sub-phases (thread 0's clock)")
for a, b, nm in sub:
    d = t[:, b] - t[:, a]
    print(f"{nm:20s} {d.mean():9.0f} cycles (p50 {np.median(d):8.0f})")

print("-- pair stage passes (thread 0)")
prev = 15
for k in [40, 41, 42, 43, 44, 45, 46, 47]:
    if t[:, k].max() > 0:
        print(f"fwd pass mark {k}: {np.mean(t[:, k] - t[:, prev]):9.0f}"); prev = k
print(f"mark 20 (len reduce) {np.mean(t[:, 20] - t[:, prev]):9.0f}"); prev = 20
for k in [48, 49, 50, 51, 52, 53, 54, 55]:
    if t[:, k].max() > 0:
        print(f"inv pass mark {k}: {np.mean(t[:, k] - t[:, prev]):9.0f}"); prev = k
print(f"mark 21 {np.mean(t[:, 21] - t[:, prev]):9.0f}"); print(f"argmax+aligned {np.mean(t[:, 23] - t[:, 21]):9.0f}")
