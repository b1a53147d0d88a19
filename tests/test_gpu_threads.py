"""Concurrent host-thread callers (SURVEY.md §8(b) "Threading"): the reference's
functions are pure and re-entrant and its distance_matrix calls align_fft from
a thread pool (proj/src/elastic.cpp:196-234), so the drop-in must give every
thread the same answer it gives a lone caller. Eight Python threads (ctypes
releases the GIL for the C-ABI calls) issue the host-buffer entry points at
once; each result must equal, bit for bit, the one a sequential call produced.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2501_17779_b200 as cva
from paper_2501_17779_b200 import synth

pytestmark = pytest.mark.gpu

THREADS = 8


def _jobs():
    jobs = []
    for t in range(THREADS):
        pts, offs, _, _ = synth.ragged_pairs(500 + t, 48, 1024)
        jobs.append(("fused", lambda pts=pts, offs=offs: cva.preprocess_align_batch(pts, offs, 1024,
                                                                                   return_aligned=True)))
        c1, c2, _, _ = synth.uniform_pairs(600 + t, 32, 256)
        jobs.append(("align", lambda c1=c1, c2=c2: cva.align_fft_batch(c1, c2, return_aligned=True)))
        s1, s2, _, _, _ = synth.srv_pairs(700 + t, 16, 512)
        jobs.append(("srv", lambda s1=s1, s2=s2: cva.srv_align_batch(s1, s2, return_aligned=True)))
        e1, e2, _, _ = synth.uniform_pairs(800 + t, 4, 64)
        p1 = np.stack([cva.preprocess(c, 64, resample=False) for c in e1])
        p2 = np.stack([cva.preprocess(c, 64, resample=False) for c in e2])
        jobs.append(("elastic", lambda p1=p1, p2=p2: cva.elastic_approach2_batch(p1, p2, return_gamma=True)))
        jobs.append(("single", lambda a=c1[0], b=c2[0]: cva.align_fft(a, b)))
        jobs.append(("energy", lambda a=p1[0], b=p2[0]: cva.elastic_energy(a, b, 0.25, 0.5, np.linspace(0, 1, 65))))
    return jobs


def _same(x, y):
    if isinstance(x, tuple):
        return all(_same(a, b) for a, b in zip(x, y))
    if isinstance(x, dict):
        return x.keys() == y.keys() and all(_same(x[k], y[k]) for k in x)
    if x is None:
        return y is None
    if isinstance(x, np.ndarray):
        if x.dtype.names:
            return all(np.array_equal(x[f], y[f], equal_nan=True) for f in x.dtype.names)
        return np.array_equal(x, y, equal_nan=True)
    if isinstance(x, float):
        return (x == y) or (np.isnan(x) and np.isnan(y))
    return x == y


def test_concurrent_host_calls_match_sequential(cuda):
    jobs = _jobs()
    seq = [fn() for _, fn in jobs]
    for rep in range(3):
        with ThreadPoolExecutor(THREADS) as ex:
            par = list(ex.map(lambda j: j[1](), jobs[::-1] if rep % 2 else jobs))
        if rep % 2:
            par = par[::-1]
        bad = [name for (name, _), a, b in zip(jobs, seq, par) if not _same(a, b)]
        assert not bad, f"concurrent results differ from sequential ones: {bad}"


def test_concurrent_errors_stay_per_thread(cuda):
    """cva_last_error is per thread: a failing call on one thread does not
    change the message or the result another thread sees."""
    c1, c2, _, _ = synth.uniform_pairs(900, 8, 128)

    def bad(_):
        with pytest.raises(ValueError):
            cva.align_fft_batch(c1[:, :100], c2)  # node count mismatch
        return True

    def good(_):
        return cva.align_fft_batch(c1, c2)[0]

    ref = good(0)
    with ThreadPoolExecutor(THREADS) as ex:
        futs = [ex.submit(bad if i % 2 else good, i) for i in range(4 * THREADS)]
        out = [f.result() for f in futs]
    for i, r in enumerate(out):
        if i % 2 == 0:
            assert _same(r, ref)
