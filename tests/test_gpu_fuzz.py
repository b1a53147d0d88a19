"""Seeded random sweep over sizes and shapes (GPU vs the oracle): raw node
counts 4..5000, output sizes 8..4096 (powers of two and not), random star
shapes with uneven node spacing, random planted shift / rotation; the fused and
split preprocess+align paths, the SRV alignment and the uniform alignment
(acceptance rule of tests/test_gpu_parity.py: shift identical up to a
documented near-tie, theta 1e-10, coordinates and energy 1e-10 relative); and
the elastic DP (bitwise the reference compiled in place, random n and slope
bound) and approach 2 (rounding-level, same iteration counts).
"""
import numpy as np
import pytest

import paper_2501_17779_b200 as cva
from test_gpu_parity import check_pair

pytestmark = pytest.mark.gpu

PI = np.pi


def star(rng, n_in, modes):
    """Closed star-shaped polygon: nodes at jittered arc positions of
    r(phi) = 1 + sum a_m cos(m phi + p_m) (node gaps between 0.2x and 1.8x the mean)."""
    a = rng.uniform(0, 0.3, modes) / np.arange(2, modes + 2)
    p = rng.uniform(0, 2 * PI, modes)
    phi = (np.arange(n_in) + rng.uniform(-0.4, 0.4, n_in)) * (2 * PI / n_in)
    r = 1 + np.sum(a[:, None] * np.cos(np.arange(2, modes + 2)[:, None] * phi[None] + p[:, None]), axis=0)
    c = np.stack([r * np.cos(phi), r * np.sin(phi)], 1)
    return c * rng.uniform(0.1, 10.0) + rng.uniform(-5, 5, 2)  # arbitrary scale and offset


def n_out_choices(rng):
    return int(rng.choice([8, 12, 64, 100, 256, 333, 512, 1000, 1024, 2048, 3000, 4096]))


@pytest.mark.parametrize("seed", range(12))
def test_random_preprocess_align(cuda, oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    n_out = n_out_choices(rng)
    pairs = 6
    curves = []
    for _ in range(pairs):
        c1 = star(rng, int(rng.integers(4, 5001)), int(rng.integers(2, 20)))
        c2 = star(rng, int(rng.integers(4, 5001)), int(rng.integers(2, 20)))
        curves += [c1, c2]
    pts, offs = cva.ragged(curves)
    res, al = cva.preprocess_align_batch(pts, offs, n_out, return_aligned=True)
    ro, ao = oracle.batch(pts, offs, n_out, mode=0, threads=4, aligned=True)
    for p in range(pairs):
        c1 = oracle.preprocess(curves[2 * p], n_out)
        c2 = oracle.preprocess(curves[2 * p + 1], n_out)
        check_pair(res[p], ro[p], c1, c2, al[p], ao[p])


@pytest.mark.parametrize("seed", range(6))
def test_random_shift_rotation_recovered(cuda, oracle, seed):
    """Same shape, start moved by k nodes and rotated: the planted (k, theta)
    is recovered and the GPU equals the oracle on the uniform path."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.choice([16, 48, 100, 256, 777, 1024, 2048, 5000]))
    base = star(rng, n, 8)
    c1 = np.stack([cva.preprocess(base, 0, resample=False)])[0]
    k = int(rng.integers(0, n))
    th = rng.uniform(-PI, PI)
    rot = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    c2 = np.roll(c1, k, axis=0) @ rot.T
    res, al = cva.align_fft_batch(c1[None], c2[None], return_aligned=True)
    want = oracle.align(c1, c2)
    assert int(res[0]["shift"]) == int(want["shift"])
    assert abs(float(res[0]["energy"])) <= 1e-12
    cth, sth = np.cos(want["theta"]), np.sin(want["theta"])
    q = c2[(np.arange(n) + int(want["shift"])) % n]
    wal = np.stack([cth * q[:, 0] + sth * q[:, 1], -sth * q[:, 0] + cth * q[:, 1]], 1)
    check_pair(res[0], want, c1, c2, al[0], wal)


@pytest.mark.parametrize("seed", range(6))
def test_random_srv_align(cuda, oracle, seed):
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.choice([8, 64, 100, 512, 1000, 2048, 4096]))
    pairs = 3
    c1 = np.stack([oracle.preprocess(star(rng, 800, 10), n) for _ in range(pairs)])
    c2 = np.stack([oracle.preprocess(star(rng, 900, 10), n) for _ in range(pairs)])
    res, alq = cva.srv_align_batch(c1, c2, return_aligned=True)
    for p in range(pairs):
        q1 = oracle.srv_center(oracle.srv_transform(c1[p]))
        q2 = oracle.srv_center(oracle.srv_transform(c2[p]))
        want = oracle.align(q1, q2)
        cth, sth = np.cos(want["theta"]), np.sin(want["theta"])
        q = q2[(np.arange(n) + int(want["shift"])) % n]
        wal = np.stack([cth * q[:, 0] + sth * q[:, 1], -sth * q[:, 0] + cth * q[:, 1]], 1)
        check_pair(res[p], want, q1, q2, alq[p], wal)


# ---------------------------------------------------------------- elastic


@pytest.mark.parametrize("seed", range(8))
def test_random_dp_bitwise(cuda, reference, seed):
    """dp_reparam on random SRV pairs (random n, slope bound, shapes, scales):
    bitwise the reference's gamma and energy."""
    ref = reference
    rng = np.random.default_rng(4000 + seed)
    n = int(rng.choice([8, 16, 24, 64, 100, 128, 200, 256, 512]))
    w = int(rng.choice([1, 2, 3, 4, 4, 4, 5]))
    pairs = 3
    q1 = np.stack([ref.srv_transform(ref.preprocess(star(rng, 600, 9), n)) for _ in range(pairs)])
    q2 = np.stack([ref.srv_transform(ref.preprocess(star(rng, 700, 9), n)) for _ in range(pairs)])
    g, e, st = cva.dp_reparam_batch(q1, q2, w)
    rg, re_, rst = ref.dp_reparam_batch(q1, q2, w)
    np.testing.assert_array_equal(st, rst)
    ok = st == 0
    np.testing.assert_array_equal(g[ok], rg[ok])
    np.testing.assert_array_equal(e[ok], re_[ok])


@pytest.mark.parametrize("seed", range(4))
def test_random_approach2(cuda, reference, seed):
    ref = reference
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.choice([32, 64, 100, 128, 256]))
    pairs = 4
    c1 = np.stack([ref.preprocess(star(rng, 500, 9), n) for _ in range(pairs)])
    c2 = np.stack([ref.preprocess(star(rng, 650, 9), n) for _ in range(pairs)])
    g = cva.elastic_approach2_batch(c1, c2)
    r = ref.elastic_approach2_batch(c1, c2)
    np.testing.assert_array_equal(g["status"], r["status"])
    np.testing.assert_allclose(g["distance"], r["distance"], rtol=1e-9, atol=1e-12)
    np.testing.assert_array_equal(g["iterations"], r["iterations"])


# Every transform plan of the pair stage (pairfft.cuh): compile-time N = 256 ..
# 2048 (fused last-forward / first-correlation pass, correlation bins kept in
# registers for the argmax), runtime N with an in-place M = 2048 plan, the
# M = 4096 kernel, and the SRV kernel with its aligned output (the raw curve 2
# brought back by TMA in the in-place plan).
@pytest.mark.parametrize("n", [256, 512, 1024, 2048, 1000, 1500, 2000])
def test_pair_stage_plans_align(cuda, oracle, n):
    rng = np.random.default_rng(5000 + n)
    pairs = 4
    c1 = np.stack([oracle.preprocess(star(rng, 700, 9), n) for _ in range(pairs)])
    c2 = np.stack([oracle.preprocess(star(rng, 800, 9), n) for _ in range(pairs)])
    res, al = cva.align_fft_batch(c1, c2, return_aligned=True)
    for p in range(pairs):
        want = oracle.align(c1[p], c2[p])
        cth, sth = np.cos(want["theta"]), np.sin(want["theta"])
        q = c2[p][(np.arange(n) + int(want["shift"])) % n]
        wal = np.stack([cth * q[:, 0] + sth * q[:, 1], -sth * q[:, 0] + cth * q[:, 1]], 1)
        check_pair(res[p], want, c1[p], c2[p], al[p], wal)


@pytest.mark.parametrize("n", [512, 1024, 2048, 1000, 1500])
@pytest.mark.parametrize("with_aligned", [True, False])
def test_pair_stage_plans_srv(cuda, oracle, n, with_aligned):
    rng = np.random.default_rng(6000 + n)
    pairs = 3
    c1 = np.stack([oracle.preprocess(star(rng, 900, 10), n) for _ in range(pairs)])
    c2 = np.stack([oracle.preprocess(star(rng, 1000, 10), n) for _ in range(pairs)])
    res, alq = cva.srv_align_batch(c1, c2, return_aligned=with_aligned)
    for p in range(pairs):
        q1 = oracle.srv_center(oracle.srv_transform(c1[p]))
        q2 = oracle.srv_center(oracle.srv_transform(c2[p]))
        want = oracle.align(q1, q2)
        cth, sth = np.cos(want["theta"]), np.sin(want["theta"])
        q = q2[(np.arange(n) + int(want["shift"])) % n]
        wal = np.stack([cth * q[:, 0] + sth * q[:, 1], -sth * q[:, 0] + cth * q[:, 1]], 1)
        if with_aligned:
            check_pair(res[p], want, q1, q2, alq[p], wal)
        else:
            check_pair(res[p], want, q1, q2)
