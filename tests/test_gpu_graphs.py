"""CUDA-graph capture of the device entry points: after one warm-up call (the
per-(device, N) twiddle table is built once, with a synchronise), the fused C1
call, the SRV alignment and the elastic batch issue only stream-ordered work,
so they can be captured into a graph and replayed; replays give bitwise the
results of eager calls."""
import numpy as np
import pytest

import paper_2501_17779_b200 as cva
from paper_2501_17779_b200 import _native, synth

pytestmark = pytest.mark.gpu


def test_graph_capture_replay_matches_eager(cuda):
    import torch

    lib = _native.load()
    pts, offs, _, _ = synth.ragged_pairs(11, 256, 1024)
    mx = int(np.diff(offs).max())
    dp, do = torch.from_numpy(pts).cuda(), torch.from_numpy(offs).cuda()
    s1, s2, _, _, _ = synth.srv_pairs(12, 64, 2048)
    d1, d2 = torch.from_numpy(s1).cuda(), torch.from_numpy(s2).cuda()
    out = torch.empty((256, 48), dtype=torch.uint8, device="cuda")
    al = torch.empty((256, 1024, 2), dtype=torch.float64, device="cuda")
    out4 = torch.empty((64, 48), dtype=torch.uint8, device="cuda")
    al4 = torch.empty_like(d2)

    def work(stream):
        _native.check(lib.cva_preprocess_align_batch(dp.data_ptr(), do.data_ptr(), 256, mx, 1024, 1,
                                                     out.data_ptr(), al.data_ptr(), stream))
        _native.check(lib.cva_srv_align_batch(d1.data_ptr(), d2.data_ptr(), 64, 2048, out4.data_ptr(),
                                              al4.data_ptr(), stream))

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        work(s.cuda_stream)  # warm-up: twiddle tables, smem attributes
    torch.cuda.synchronize()
    eager = [t.clone() for t in (out, al, out4, al4)]
    for t in (out, al, out4, al4):
        t.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        work(s.cuda_stream)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, (out, al, out4, al4)):
        assert torch.equal(a, b)
    res = cva.decode_results(out)
    assert (res["status"] == 0).all()
