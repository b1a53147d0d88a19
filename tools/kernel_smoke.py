"""Small invocations of every kernel family (fused C1, split preprocess/align,
all-pairs, four-step and radix-16 large N, SRV at both transform layouts,
elastic approach 1/2 and the DP) in one process, for quick bring-up checks:

    python tools/kernel_smoke.py [all|c1|c2|c3|c4|elastic]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_17779_b200 as cva  # noqa: E402
from paper_2501_17779_b200 import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "c1"):
    pts, offs, _, _ = synth.ragged_pairs(3, 4, 1024)
    r, a = cva.preprocess_align_batch(pts, offs, 1024, return_aligned=True)
    assert (r["status"] == 0).all()
    prep, st = cva.preprocess_batch(pts, offs, 512)
    r2, _ = cva.align_fft_batch(prep[0::2], prep[1::2], return_aligned=True)
if which in ("all", "c2"):
    pts, offs = synth.ragged_curves(5, 6)
    prep, _ = cva.preprocess_batch(pts, offs, 512)
    cva.allpairs(prep)
if which in ("all", "c3"):
    c1, c2, _, _ = synth.uniform_pairs(7, 2, 16384)
    cva.preprocess_align_uniform(c1, c2, return_aligned=True)
    c1, c2, _, _ = synth.uniform_pairs(7, 2, 4097)
    cva.align_fft_batch(c1, c2)
if which in ("all", "c4"):
    s1, s2, _, _, _ = synth.srv_pairs(9, 3, 2048)
    cva.srv_align_batch(s1, s2, return_aligned=True)
    s1, s2, _, _, _ = synth.srv_pairs(9, 3, 512)
    cva.srv_align_batch(s1, s2, return_aligned=True)
if which in ("all", "elastic"):
    pts, offs = synth.ragged_curves(11, 3)
    prep, _ = cva.preprocess_batch(pts, offs, 64)
    cva.elastic_distance_matrix(prep)
    cva.elastic_distance_matrix(prep, method=1)
    q = np.ascontiguousarray(prep[:2])
    cva.dp_reparam_batch(q, q[::-1].copy())
torch.cuda.synchronize() if torch.cuda.is_available() else None
print("ok")
