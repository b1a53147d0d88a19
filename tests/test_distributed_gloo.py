"""CPU, world_size 2 over gloo: the multi-GPU host logic (pair / row sharding,
padded all-gather, assembly) with the CPU oracle standing in for the per-rank
kernel. The GPU kernels themselves are covered by tests/test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2501_17779_b200.distributed import shard_range


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("count,world", [(0, 2), (1, 2), (5, 2), (7, 3), (4096, 8), (2048, 8), (13, 4)])
def test_shard_range_partitions(count, world):
    spans = [shard_range(count, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == count
    for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
        assert e0 == b1
    sizes = [e - b for b, e in spans]
    assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, root, q):
    import sys

    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch.distributed as dist

    from paper_2501_17779_b200 import distributed as D
    from pyoracle import Oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = Oracle()
        rng = np.random.default_rng(0)
        m, n = 7, 32
        curves = rng.uniform(-1, 1, (m, n, 2))

        def rows(c, rb, re):
            e = np.zeros((re - rb, m))
            k = np.zeros((re - rb, m), dtype=np.int32)
            t = np.zeros((re - rb, m))
            for i in range(rb, re):
                for j in range(m):
                    r = O.align(c[i], c[j])
                    e[i - rb, j], k[i - rb, j], t[i - rb, j] = r["energy"], r["shift"], r["theta"]
            return e, k, t

        e, k, t = D.allpairs_distributed(curves, compute=rows)
        c1 = rng.uniform(-1, 1, (5, n, 2))
        c2 = rng.uniform(-1, 1, (5, n, 2))

        def pairs(a, b):
            return np.array([O.align(x, y) for x, y in zip(a, b)])

        res, span = D.align_sharded(c1, c2, compute=pairs)
        q.put((rank, e.numpy(), k.numpy(), t.numpy(), res.tobytes(), span))
    finally:
        dist.destroy_process_group()


def test_allpairs_and_pairs_gather_world2():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, root, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda x: x[0])
    import sys

    sys.path.insert(0, os.path.join(root, "oracle"))
    from pyoracle import ALIGNMENT_DTYPE, Oracle

    O = Oracle()
    rng = np.random.default_rng(0)
    curves = rng.uniform(-1, 1, (7, 32, 2))
    c1 = rng.uniform(-1, 1, (5, 32, 2))
    c2 = rng.uniform(-1, 1, (5, 32, 2))
    for rank, e, k, t, res, span in outs:
        assert e.shape == (7, 7)
        for i in range(7):
            for j in range(7):
                r = O.align(curves[i], curves[j])
                assert k[i, j] == r["shift"] and e[i, j] == r["energy"] and t[i, j] == r["theta"]
        full = np.frombuffer(res, dtype=ALIGNMENT_DTYPE)
        assert len(full) == 5
        for p in range(5):
            assert full[p]["shift"] == O.align(c1[p], c2[p])["shift"]
    assert outs[0][5] == (0, 3) and outs[1][5] == (3, 5)
