"""Multi-GPU sharding of the alignment path (one process per GPU, torch.distributed).

SURVEY.md §8(e): pairs are independent, so batches (C1 / C3 / C4) are split by
contiguous pair ranges with no data-path collective; the all-pairs matrix (C2)
is split by row blocks, each rank recomputes every curve's spectrum locally
(cheaper than exchanging them) and the row blocks are gathered to the
destination with one collective (``all_gather_into_tensor`` on NCCL, which
moves each rank's block once over NVLink/NVSwitch).

Every function takes an optional ``compute`` callable so the host logic (ranges,
padding, gather, assembly) can be exercised on CPU with the gloo backend and a
CPU stand-in for the per-rank kernel (tests/test_distributed_gloo.py); on GPUs
the default is the CUDA library.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) of `count` items for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(count, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def _world(group):
    return dist.get_rank(group), dist.get_world_size(group)


def align_sharded(c1, c2, group=None, compute=None, gather: bool = True):
    """Align this rank's contiguous share of the pairs (c1[i], c2[i]).

    c1, c2: the full batch (numpy or tensors, identical on all ranks) — each rank
    touches only its slice. Returns (results of this rank's slice, (begin, end)),
    or with gather=True the full structured result array on every rank.
    """
    from . import api

    rank, world = _world(group)
    b, e = shard_range(len(c1), rank, world)
    compute = compute or (lambda a, b_: api.align_fft_batch(a, b_)[0])
    part = np.asarray(compute(c1[b:e], c2[b:e]))
    if not gather:
        return part, (b, e)
    raw = np.frombuffer(np.ascontiguousarray(part).tobytes(), dtype=np.uint8).reshape(-1, 48)
    full = _all_gather_rows(torch.from_numpy(raw.copy()), len(c1), group)
    return np.frombuffer(full.numpy().tobytes(), dtype=part.dtype), (b, e)


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


def allpairs_distributed(curves, group=None, compute=None):
    """C2: every rank computes rows [begin, end) of the all-pairs matrices of the
    (preprocessed, identical on all ranks) curves and the blocks are gathered on
    all ranks. Returns (energy, shift, theta) as tensors on the curves' device."""
    from . import api

    rank, world = _world(group)
    count = curves.shape[0]
    b, e = shard_range(count, rank, world)
    compute = compute or (lambda c, rb, re: api.allpairs(c, rb, re))
    en, sh, th = compute(curves, b, e)
    en, sh, th = (torch.as_tensor(x) for x in (en, sh, th))
    return (_all_gather_rows(en, count, group), _all_gather_rows(sh, count, group),
            _all_gather_rows(th, count, group))
