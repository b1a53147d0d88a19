"""Time cva_align_batch (device buffers, CUDA events) for 4096 pairs at several N.

    python tools/time_n.py [N ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_17779_b200 import _native  # noqa: E402

lib = _native.load()
for n in [int(x) for x in sys.argv[1:]] or [1000, 1024, 1500, 2000, 2048, 4096]:
    P = 4096
    rng = np.random.default_rng(n)
    a = torch.from_numpy(rng.uniform(-1, 1, (P, n, 2))).cuda()
    b = torch.from_numpy(rng.uniform(-1, 1, (P, n, 2))).cuda()
    out = torch.empty((P, 48), dtype=torch.uint8, device="cuda")
    al = torch.empty_like(b)
    s = torch.cuda.current_stream().cuda_stream

    def f():
        _native.check(lib.cva_align_batch(a.data_ptr(), b.data_ptr(), P, n, out.data_ptr(), al.data_ptr(), s))

    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"N={n:6d}  {e0.elapsed_time(e1) / 10 * 1e3:9.1f} us per 4096 pairs")
