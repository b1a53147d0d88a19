"""GPU: the multi-GPU host logic on NCCL with the default (CUDA library)
compute, world size 1 on the one device of the box: align_sharded on CUDA
tensors and on numpy input, and the C2 chunked gather (AllPairsGather) against
the single-call all-pairs kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2501_17779_b200 as cva
from paper_2501_17779_b200 import distributed as D
from paper_2501_17779_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group(cuda):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_align_sharded_nccl_default_compute(nccl_group):
    c1, c2, _, _ = synth.uniform_pairs(3, 37, 256)
    ref, _ = cva.align_fft_batch(c1, c2)
    got, span = D.align_sharded(c1, c2)  # numpy in: structured array out
    assert span == (0, 37)
    assert np.array_equal(got["shift"], ref["shift"]) and np.array_equal(got["theta"], ref["theta"])
    d1, d2 = torch.from_numpy(c1).cuda(), torch.from_numpy(c2).cuda()
    gt, _ = D.align_sharded(d1, d2)  # CUDA in: device uint8 records out
    assert gt.is_cuda and gt.shape == (37, 48)
    dec = cva.decode_results(gt.cpu())
    assert np.array_equal(dec["shift"], ref["shift"]) and np.array_equal(dec["energy"], ref["energy"])


def test_allpairs_gather_nccl_matches_single_call(nccl_group):
    pts, offs = synth.ragged_curves(5, 64)
    prep, st = cva.preprocess_batch(pts, offs, 128)
    assert (st == 0).all()
    dprep = torch.from_numpy(prep).cuda()
    e0, k0, t0 = cva.allpairs(dprep)
    from paper_2501_17779_b200 import _native

    lib = _native.load()
    s = torch.cuda.current_stream().cuda_stream

    def fill(rb, re, e, k, th):
        _native.check(lib.cva_allpairs(dprep.data_ptr(), 64, 128, rb, re, e.data_ptr(), k.data_ptr(),
                                       th.data_ptr(), s))

    g = D.AllPairsGather(64, fill, chunks=3, dst=0)
    g.run()
    e, k, t = g.assemble()
    torch.cuda.synchronize()
    assert torch.equal(e, e0) and torch.equal(k, k0) and torch.equal(t, t0)
