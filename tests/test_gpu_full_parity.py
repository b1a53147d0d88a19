"""GPU, full size: every pair of the bench's C1 batch (4096, the bench's seed),
2048 C4 pairs, all 256 C3 pairs at N = 65536 and 16 full rows of the C2 matrix
(32768 cells), each checked against the reference's own sources compiled in
place (oracle/_ref) with the acceptance rule of tests/parity_rule.py
(SURVEY.md §8(c)); plus the oracle pins (tests/test_oracle_pins.py) run inside
the GPU job, so the chain GPU -> oracle -> reference is in the GPU record.
The CPU side runs on all host threads (about a second per config)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2501_17779_b200 as cva
from paper_2501_17779_b200 import synth
from parity_rule import compare, ragged_of_pairs

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1
BENCH_SEED = 1  # bench.py --seed default


def _ok(summary):
    assert summary["violations"] == 0, summary
    assert summary["status_ok"] == summary["pairs"], summary
    assert summary["shift_equal"] + summary["near_ties"] == summary["pairs"], summary


def test_c1_every_pair_vs_reference(cuda, reference):
    cfg = synth.CONFIGS["c1"]
    pts, offs, _, _ = synth.ragged_pairs(BENCH_SEED, cfg["pairs"], cfg["N"])
    res, al = cva.preprocess_align_batch(pts, offs, cfg["N"], return_aligned=True)
    ro, ao = reference.batch(pts, offs, cfg["N"], mode=0, threads=THREADS, aligned=True)
    prep, _ = cva.preprocess_batch(pts, offs, cfg["N"])
    s = compare(res, ro, al, ao, prep[0::2], prep[1::2])
    _ok(s)
    assert s["max_dtheta"] < 1e-12 and s["max_coord_rel"] < 1e-11


def test_c4_2048_pairs_vs_reference(cuda, reference):
    P, N = 2048, synth.CONFIGS["c4"]["N"]
    c1, c2, _, _, _ = synth.srv_pairs(BENCH_SEED, P, N)
    res, alq = cva.srv_align_batch(c1, c2, return_aligned=True)
    pts, offs = ragged_of_pairs(c1, c2)
    ro, ao = reference.batch(pts, offs, N, mode=2, threads=THREADS, aligned=True)
    q1 = np.stack([reference.srv_center(reference.srv_transform(c1[p])) for p in range(P)])
    q2 = np.stack([reference.srv_center(reference.srv_transform(c2[p])) for p in range(P)])
    _ok(compare(res, ro, alq, ao, q1, q2))


def test_c3_all_256_pairs_vs_reference(cuda, reference):
    cfg = synth.CONFIGS["c3"]
    c1, c2, _, _ = synth.uniform_pairs(BENCH_SEED, cfg["pairs"], cfg["N"], cfg["modes"], cfg["amp"],
                                       cfg["amp_exp"], cfg["sigma"])
    res, al = cva.preprocess_align_uniform(c1, c2, return_aligned=True)
    pts, offs = ragged_of_pairs(c1, c2)
    ro, ao = reference.batch(pts, offs, cfg["N"], mode=0, resample=False, threads=THREADS, aligned=True)
    u = np.stack([reference.preprocess(c1[p], 0, resample=False) for p in range(cfg["pairs"])])
    v = np.stack([reference.preprocess(c2[p], 0, resample=False) for p in range(cfg["pairs"])])
    _ok(compare(res, ro, al, ao, u, v))


def test_c2_16_full_rows_vs_reference(cuda, reference):
    cfg = synth.CONFIGS["c2"]
    M, N = cfg["curves"], cfg["N"]
    pts, offs = synth.ragged_curves(BENCH_SEED, M)
    prep, st = cva.preprocess_batch(pts, offs, N)
    assert (st == 0).all()
    e, k, th = cva.allpairs(prep)
    rows = np.linspace(0, M - 1, 16).astype(int)
    firsts = np.repeat(prep[rows], M, axis=0)
    seconds = np.tile(prep, (len(rows), 1, 1))
    a_pts, a_offs = ragged_of_pairs(firsts, seconds)
    ro, _ = reference.batch(a_pts, a_offs, N, mode=1, resample=False, threads=THREADS)
    g = np.zeros(len(rows) * M, dtype=ro.dtype)
    g["shift"], g["theta"], g["energy"] = k[rows].ravel(), th[rows].ravel(), e[rows].ravel()
    g["trace"], g["t0"] = ro["trace"], k[rows].ravel() / N
    _ok(compare(g, ro, None, None, firsts, seconds))
    # the matrices' rows are the same cells as the pair kernel (spectrum reuse changes nothing)
    assert np.allclose(np.diag(e), 0.0, atol=1e-14)


def test_oracle_pins_in_gpu_job():
    """tests/test_oracle_pins.py (C oracle == reference compiled in place, bit
    for bit, on the golden fixtures and live batches), run here so the GPU
    record carries the whole parity chain."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_oracle_pins.py")], capture_output=True, text=True,
                       cwd=root, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout and "skipped" not in p.stdout.splitlines()[-1], p.stdout[-500:]
