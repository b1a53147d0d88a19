"""Multi-GPU sharding of the alignment path (one process per GPU, torch.distributed).

SURVEY.md §8(e): pairs are independent, so batches (C1 / C3 / C4) are split by
contiguous pair ranges with no data-path collective; the all-pairs matrix (C2)
is split by row blocks, each rank recomputes every curve's spectrum locally
(cheaper than exchanging 16.8 MB of spectra) and the row blocks travel to the
destination rank with one gather per row chunk (packed 20-byte cells), issued
asynchronously so the transfer of chunk c overlaps the computation of chunk
c + 1 (the pair-parallel pattern of the reference's thread pool,
proj/src/elastic.cpp:196-234, one level up).

Every function takes an optional ``compute`` callable so the host logic
(ranges, padding, gathers, assembly) can be exercised on CPU with the gloo
backend and a CPU stand-in for the per-rank kernel
(tests/test_distributed_gloo.py); on GPUs the default is the CUDA library and
the collectives run on NCCL with device tensors.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

CELL_BYTES = 20  # energy f64 + theta f64 + shift i32 per all-pairs cell


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) of `count` items for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(count, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def _world(group):
    return dist.get_rank(group), dist.get_world_size(group)


def collective_device(group=None) -> torch.device:
    """Where this group's collectives take their tensors: the current CUDA device
    for NCCL, the host for gloo."""
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def align_sharded(c1, c2, group=None, compute=None, gather: bool = True):
    """Align this rank's contiguous share of the pairs (c1[i], c2[i]).

    c1, c2: the full batch (numpy or CUDA tensors, identical on all ranks) -
    each rank touches only its slice. Returns (this rank's results, (begin,
    end)), or with gather=True all results on every rank: a structured numpy
    array for numpy input, a ``(pairs, 48)`` uint8 tensor on the input's device
    for CUDA input (decode with ``api.decode_results``).
    """
    from . import api

    rank, world = _world(group)
    b, e = shard_range(len(c1), rank, world)
    compute = compute or (lambda a, b_: api.align_fft_batch(a, b_)[0])
    part = compute(c1[b:e], c2[b:e])
    if not gather:
        return part, (b, e)
    dev = collective_device(group)
    if isinstance(part, torch.Tensor):
        block = part.reshape(-1).view(torch.uint8).reshape(-1, 48)
        full = _all_gather_rows(block.to(dev), len(c1), group)
        return full.to(part.device), (b, e)
    part = np.ascontiguousarray(part)
    raw = np.frombuffer(part.tobytes(), dtype=np.uint8).reshape(-1, 48)
    full = _all_gather_rows(torch.from_numpy(raw.copy()).to(dev), len(c1), group)
    return np.frombuffer(full.cpu().numpy().tobytes(), dtype=part.dtype), (b, e)


def _all_gather_rows(block: torch.Tensor, total_rows: int, group=None) -> torch.Tensor:
    """Concatenate each rank's row block (rank order) on every rank. Blocks are
    padded to the largest share so one all_gather_into_tensor suffices."""
    rank, world = _world(group)
    shares = [shard_range(total_rows, r, world) for r in range(world)]
    width = max(e - b for b, e in shares)
    padded = torch.zeros((width,) + tuple(block.shape[1:]), dtype=block.dtype, device=block.device)
    padded[: block.shape[0]] = block
    out = torch.empty((world * width,) + tuple(block.shape[1:]), dtype=block.dtype, device=block.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    return torch.cat([out[r * width: r * width + (e - b)] for r, (b, e) in enumerate(shares)])


def _cell_views(buf: torch.Tensor, rows_cap: int, count: int, rows: int):
    """energy / shift / theta views of one packed chunk buffer (struct of arrays:
    energy f64 [rows_cap x count], theta f64 [...], shift i32 [...]); the first
    `rows` rows are used."""
    n8 = rows_cap * count * 8
    e = buf[:n8].view(torch.float64)[: rows * count].view(rows, count)
    th = buf[n8: 2 * n8].view(torch.float64)[: rows * count].view(rows, count)
    k = buf[2 * n8: 2 * n8 + rows_cap * count * 4].view(torch.int32)[: rows * count].view(rows, count)
    return e, k, th


class AllPairsGather:
    """C2 over a process group: rows of the count x count matrices sharded by
    `shard_range`, each rank's block computed in `chunks` row chunks, chunk c
    packed (20 B/cell) in one buffer and gathered to `dst` with one async
    gather, overlapping chunk c + 1's computation. Buffers are allocated once
    (the bench reuses the object every step).

    compute(rb, re, energy, shift, theta): fill rows [rb, re) into the views
    (float64 / int32 / float64, (re - rb) x count) on the collective device,
    stream-ordered before the gather is issued.
    """

    def __init__(self, count: int, compute, group=None, chunks: int = 4, dst: int = 0):
        self.group, self.dst, self.count, self.compute = group, dst, count, compute
        self.rank, self.world = _world(group)
        self.shares = [shard_range(count, r, self.world) for r in range(self.world)]
        width = max(e - b for b, e in self.shares)
        self.chunks = max(1, min(chunks, width)) if width else 1
        self.crow = max(1, math.ceil(width / self.chunks))
        dev = collective_device(group)
        self.nbytes = (CELL_BYTES * self.crow * count + 255) // 256 * 256  # 256-B aligned chunks
        self.send = torch.zeros((self.chunks, self.nbytes), dtype=torch.uint8, device=dev)
        self.recv = (torch.zeros((self.world, self.chunks, self.nbytes), dtype=torch.uint8, device=dev)
                     if self.rank == dst else None)

    def _rows(self, r: int, c: int) -> tuple[int, int]:
        b, e = self.shares[r]
        rb = b + c * self.crow
        return rb, max(rb, min(e, rb + self.crow))

    def run(self) -> None:
        """Compute this rank's rows and gather them to dst (returns once every
        gather is complete / stream-ordered: NCCL work is waited on the
        current stream)."""
        works = []
        for c in range(self.chunks):
            rb, re = self._rows(self.rank, c)
            if re > rb:
                self.compute(rb, re, *_cell_views(self.send[c], self.crow, self.count, re - rb))
            gl = [self.recv[r, c] for r in range(self.world)] if self.rank == self.dst else None
            works.append(dist.gather(self.send[c], gather_list=gl, dst=self.dst, group=self.group, async_op=True))
        for w in works:
            w.wait()

    def assemble(self):
        """On dst: the (energy, shift, theta) matrices from the gathered chunks;
        None elsewhere."""
        if self.rank != self.dst:
            return None
        dev = self.recv.device
        en = torch.empty((self.count, self.count), dtype=torch.float64, device=dev)
        sh = torch.empty((self.count, self.count), dtype=torch.int32, device=dev)
        th = torch.empty((self.count, self.count), dtype=torch.float64, device=dev)
        for r in range(self.world):
            for c in range(self.chunks):
                rb, re = self._rows(r, c)
                if re > rb:
                    e, k, t = _cell_views(self.recv[r, c], self.crow, self.count, re - rb)
                    en[rb:re], sh[rb:re], th[rb:re] = e, k, t
        return en, sh, th


def allpairs_distributed(curves, group=None, compute=None, chunks: int = 4, dst: int | None = None):
    """C2: rows sharded over the group, gathered to `dst` (one gather per row
    chunk, see AllPairsGather). dst=None: every rank gets the matrices (the
    gathered ones are broadcast from rank 0). Returns (energy, shift, theta)
    tensors on the collective device (None on non-destination ranks).

    compute(curves, rb, re) -> (energy, shift, theta) of rows [rb, re); the
    default is the CUDA library (``api.allpairs``)."""
    from . import api

    count = curves.shape[0]
    compute = compute or (lambda c, rb, re: api.allpairs(c, rb, re))

    def fill(rb, re, e, k, th):
        en, sh, t = compute(curves, rb, re)
        e.copy_(torch.as_tensor(en).to(e.device))
        k.copy_(torch.as_tensor(sh).to(k.device).to(torch.int32))
        th.copy_(torch.as_tensor(t).to(th.device))

    g = AllPairsGather(count, fill, group=group, chunks=chunks, dst=0 if dst is None else dst)
    g.run()
    out = g.assemble()
    if dst is not None:
        return out
    dev = collective_device(group)
    if out is None:
        out = (torch.empty((count, count), dtype=torch.float64, device=dev),
               torch.empty((count, count), dtype=torch.int32, device=dev),
               torch.empty((count, count), dtype=torch.float64, device=dev))
    for x in out:
        dist.broadcast(x, src=0, group=group)
    return out
