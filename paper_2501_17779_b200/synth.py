"""Seeded synthetic workloads for the BASELINE.json configs (harness; see csrc/synth.cpp).

Every array is float64 (x, y) interleaved; ragged batches come with int64 offsets.
"""
from __future__ import annotations

import os

import numpy as np

from ._native import load_synth

_THREADS = max(1, min(32, os.cpu_count() or 1))

# name -> generator parameters (BASELINE.json "configs")
CONFIGS = {
    "c0": dict(pairs=1, N=256, modes=7, amp=0.3, amp_exp=1.0, sigma=1e-3),
    "c1": dict(pairs=4096, N=1024, modes=16, amp=0.3, amp_exp=1.0, sigma=1e-3, n_min=300, n_max=3000),
    "c2": dict(curves=2048, N=512, modes=16, amp=0.3, amp_exp=1.0, n_min=300, n_max=3000),
    "c3": dict(pairs=256, N=65536, modes=64, amp=0.3, amp_exp=1.5, sigma=1e-4),
    "c4": dict(pairs=8192, N=2048, modes=16, amp=0.3, amp_exp=1.0),
    # elastic distance matrix (approach 2): all ordered pairs of
    # `curves` C2-generator curves preprocessed to N (distance_matrix(curves, approach2, N))
    "e1": dict(curves=64, N=256, modes=16, amp=0.3, amp_exp=1.0, n_min=300, n_max=3000),
}


def _p(a):
    return a.ctypes.data if a is not None else 0


def ragged_pairs(seed, pairs, N, modes=16, amp=0.3, amp_exp=1.0, sigma=1e-3, n_min=300, n_max=3000):
    """C1: raw pairs with n_in ~ U{n_min..n_max}. Returns (points, offsets, k, theta)."""
    lib = load_synth()
    offs = np.zeros(2 * pairs + 1, dtype=np.int64)
    assert lib.cva_synth_sizes(seed, 2 * pairs, n_min, n_max, _p(offs)) == 0
    pts = np.empty((int(offs[-1]), 2), dtype=np.float64)
    k = np.empty(pairs, dtype=np.int64)
    th = np.empty(pairs, dtype=np.float64)
    assert lib.cva_synth_ragged_pairs(seed, pairs, N, modes, amp, amp_exp, sigma, _p(offs), _p(pts),
                                      _p(k), _p(th), _THREADS) == 0
    return pts, offs, k, th


def ragged_curves(seed, curves, modes=16, amp=0.3, amp_exp=1.0, n_min=300, n_max=3000):
    """C2: independent raw curves. Returns (points, offsets)."""
    lib = load_synth()
    offs = np.zeros(curves + 1, dtype=np.int64)
    assert lib.cva_synth_sizes(seed ^ 0x5EED, curves, n_min, n_max, _p(offs)) == 0
    pts = np.empty((int(offs[-1]), 2), dtype=np.float64)
    assert lib.cva_synth_ragged_curves(seed, curves, modes, amp, amp_exp, _p(offs), _p(pts), _THREADS) == 0
    return pts, offs


def uniform_pairs(seed, pairs, N, modes=7, amp=0.3, amp_exp=1.0, sigma=1e-3):
    """C0 / C3: uniformly sampled pairs. Returns (c1, c2, k, theta), c* (pairs, N, 2)."""
    lib = load_synth()
    c1 = np.empty((pairs, N, 2), dtype=np.float64)
    c2 = np.empty((pairs, N, 2), dtype=np.float64)
    k = np.empty(pairs, dtype=np.int64)
    th = np.empty(pairs, dtype=np.float64)
    assert lib.cva_synth_uniform_pairs(seed, pairs, N, modes, amp, amp_exp, sigma, _p(c1), _p(c2),
                                       _p(k), _p(th), _THREADS) == 0
    return c1, c2, k, th


def srv_pairs(seed, pairs, N, modes=16, amp=0.3, amp_exp=1.0):
    """C4: (c1, c2, k, theta, u) with c2 = rot(c1(gamma(t) - k/N)), gamma = t + 0.05 u sin(2 pi t)."""
    lib = load_synth()
    c1 = np.empty((pairs, N, 2), dtype=np.float64)
    c2 = np.empty((pairs, N, 2), dtype=np.float64)
    k = np.empty(pairs, dtype=np.int64)
    th = np.empty(pairs, dtype=np.float64)
    u = np.empty(pairs, dtype=np.float64)
    assert lib.cva_synth_srv_pairs(seed, pairs, N, modes, amp, amp_exp, _p(c1), _p(c2), _p(k), _p(th),
                                   _p(u), _THREADS) == 0
    return c1, c2, k, th, u
