"""GPU parity for the elastic (SRV) matching rows — SURVEY.md 8(f) rows 2-3:
batched dp_reparam (proj/src/srv.cpp:180-257) and elastic_distance_approach2
(proj/src/elastic.cpp:102-174) / distance_matrix (:176-236), through the C ABI,
against the reference's own code compiled in place (oracle/_ref).

Acceptance rule:
  * dp_reparam: bitwise equal gamma and energy for the same SRV inputs (the GPU
    restates dp_step_cost and the recurrence operation for operation);
  * approach 2: the GPU's rigid steps use the FFT pair stage (rotation within
    ulps of the reference's SVD) and CUDA cos/sin (<= 2 ulp), so the search
    agrees to rounding: distance within 1e-8 relative (+1e-12 absolute),
    identical iteration count and convergence flag, and the properties the
    reference's own tests assert (test_elastic.cpp, acceptance.cpp:455-530).
"""
import numpy as np
import pytest

import paper_2501_17779_b200 as cva

pytestmark = pytest.mark.gpu

FAM = ["circle", "superellipse", "hippopede", "bumps", "limacon", "clover", "fourier_random"]
DIST_RTOL = 1e-8


def prep(reference, family, n, seed=1, n_raw=512):
    return reference.preprocess(reference.gen_curve(family, n_raw, seed=seed), n, True)


def srv_pair(reference, n, seed):
    a = prep(reference, "fourier_random", n, seed)
    b = prep(reference, "fourier_random", n, seed + 100)
    return reference.srv_transform(a), reference.srv_transform(b)


# ------------------------------------------------------------------- DP


@pytest.mark.parametrize("n", [8, 16, 48, 64, 100, 128, 256])
def test_dp_bitwise_vs_reference(cuda, reference, n):
    pairs = [srv_pair(reference, n, s) for s in range(1, 5)]
    q1 = np.stack([p[0] for p in pairs])
    q2 = np.stack([p[1] for p in pairs])
    g, e, st = cva.dp_reparam_batch(q1, q2)
    rg, re_, rst = reference.dp_reparam_batch(q1, q2)
    assert (st == 0).all() and (rst == 0).all()
    np.testing.assert_array_equal(g, rg)
    np.testing.assert_array_equal(e, re_)


@pytest.mark.parametrize("w", [1, 2, 3, 5])
def test_dp_other_slopes_bitwise(cuda, reference, w):
    q1, q2 = srv_pair(reference, 64, 7)
    g, e, st = cva.dp_reparam_batch(q1[None], q2[None], max_slope=w)
    rg, re_, rst = reference.dp_reparam_batch(q1[None], q2[None], max_slope=w)
    assert st[0] == rst[0] == 0
    np.testing.assert_array_equal(g, rg)
    np.testing.assert_array_equal(e, re_)


def test_dp_identity_for_identical_curves(cuda, reference):  # test_srv.cpp:190-198
    q = reference.srv_transform(prep(reference, "bumps", 64))
    g, e = cva.dp_reparam(q, q)
    np.testing.assert_allclose(g, np.arange(65) / 64, atol=1e-12)
    assert e == pytest.approx(0.0, abs=1e-12)


def test_dp_valid_warps_and_energy_bound(cuda, reference):  # test_srv.cpp:200-230, acceptance.cpp:483-497
    q1 = np.stack([srv_pair(reference, 48, s)[0] for s in range(1, 21)])
    q2 = np.stack([srv_pair(reference, 48, s)[1] for s in range(1, 21)])
    g, e, st = cva.dp_reparam_batch(q1, q2)
    assert (st == 0).all()
    assert (g[:, 0] == 0).all() and (g[:, -1] == 1).all()
    assert (np.diff(g, axis=1) >= 0).all()
    ident = np.arange(49) / 48
    for p in range(20):
        e_id = reference.elastic_energy(q1[p], q2[p], 0.0, 0.0, ident)
        assert e[p] <= e_id + 1e-12


def test_dp_device_tensors(cuda, reference):
    import torch

    q1, q2 = srv_pair(reference, 128, 3)
    g, e, st = cva.dp_reparam_batch(torch.from_numpy(q1[None]).cuda(), torch.from_numpy(q2[None]).cuda())
    torch.cuda.synchronize()
    rg, re_, _ = reference.dp_reparam_batch(q1[None], q2[None])
    np.testing.assert_array_equal(g.cpu().numpy(), rg)
    np.testing.assert_array_equal(e.cpu().numpy(), re_)


# ---------------------------------------------------------------- approach 2


def _pairs(reference, n, count, seed0=1):
    c1, c2 = [], []
    for k in range(count):
        c1.append(prep(reference, FAM[k % len(FAM)], n, seed0 + k))
        c2.append(prep(reference, FAM[(k + 3) % len(FAM)], n, seed0 + 50 + k))
    return np.stack(c1), np.stack(c2)


def _check_vs_reference(g, r):
    assert (g["status"] == 0).all() and (r["status"] == 0).all()
    np.testing.assert_allclose(g["distance"], r["distance"], rtol=DIST_RTOL, atol=1e-12)
    np.testing.assert_allclose(g["energy"], r["energy"], rtol=2 * DIST_RTOL, atol=1e-12)
    np.testing.assert_array_equal(g["iterations"], r["iterations"])
    np.testing.assert_array_equal(g["converged"], r["converged"])


@pytest.mark.parametrize("n", [64, 128])
def test_approach2_matches_reference(cuda, reference, n):
    c1, c2 = _pairs(reference, n, 8)
    g = cva.elastic_approach2_batch(c1, c2, return_gamma=True)
    r = reference.elastic_approach2_batch(c1, c2, threads=8, gamma=True)
    _check_vs_reference(g, r)
    # energy trace (ElasticMatch::energy_trace, elastic.cpp:119, :160): same length, same values
    # to rounding, never increasing (acceptance.cpp:463-470)
    np.testing.assert_array_equal(np.isnan(g["energy_trace"]), np.isnan(r["energy_trace"]))
    np.testing.assert_allclose(g["energy_trace"], r["energy_trace"], rtol=2 * DIST_RTOL, atol=1e-12)
    t = g["energy_trace"]
    assert np.all(np.nan_to_num(np.diff(t, axis=1), nan=-1.0) <= 1e-12)
    np.testing.assert_allclose(g["t0"], r["t0"], atol=1e-9)
    # gamma: a valid warp in every pair (srv.cpp:58-69)
    assert (g["gamma"][:, 0] == 0).all() and (g["gamma"][:, -1] == 1).all()
    assert (np.diff(g["gamma"], axis=1) >= -1e-12).all()


def test_approach2_n256_matches_reference(cuda, reference):
    c1, c2 = _pairs(reference, 256, 4, seed0=11)
    _check_vs_reference(cva.elastic_approach2_batch(c1, c2), reference.elastic_approach2_batch(c1, c2, threads=4))


def test_approach2_non_power_of_two(cuda, reference):
    c1, c2 = _pairs(reference, 100, 4, seed0=21)
    _check_vs_reference(cva.elastic_approach2_batch(c1, c2), reference.elastic_approach2_batch(c1, c2, threads=4))


def test_approach2_identical_curves(cuda, reference):  # test_elastic.cpp:35-40
    c = prep(reference, "clover", 64)
    m = cva.elastic_distance_approach2(c, c)
    assert m.distance < 1e-6 and m.converged


def test_approach2_orbit_invariance(cuda, reference):  # acceptance.cpp:514-524
    for n in (128, 256):
        c1 = prep(reference, "limacon", n)
        k = n // 3
        th = 1.234
        rot = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        c2 = np.roll(c1, -k, axis=0) @ rot.T
        m = cva.elastic_distance_approach2(c1, c2)
        assert m.distance <= 0.005, m.distance


def test_approach2_energy_is_realised(cuda, reference):
    """The returned state reproduces the returned energy (elastic_energy with
    the reference's own code on the GPU's t0, theta, gamma) and distance = sqrt."""
    c1, c2 = _pairs(reference, 64, 4, seed0=31)
    g = cva.elastic_approach2_batch(c1, c2, return_gamma=True)
    for p in range(4):
        q1, q2 = reference.srv_transform(c1[p]), reference.srv_transform(c2[p])
        e = reference.elastic_energy(q1, q2, g["t0"][p], g["theta"][p], g["gamma"][p])
        assert e == pytest.approx(g["energy"][p], rel=1e-12, abs=1e-15)
        assert g["distance"][p] == pytest.approx(np.sqrt(g["energy"][p]), rel=1e-15)


def test_distance_matrix_matches_reference(cuda, reference):  # test_elastic.cpp:113-135
    raw = np.stack([reference.gen_curve(FAM[k], 400, seed=k + 1) for k in range(5)])
    d = cva.distance_matrix(list(raw), 64)  # GPU preprocess + GPU matching
    rd = reference.distance_matrix_approach2(raw, 64, threads=8)
    np.testing.assert_allclose(d, rd, rtol=DIST_RTOL, atol=1e-12)
    assert np.allclose(np.diag(d), 0.0, atol=1e-6)


def test_distance_matrix_equals_pair_batch(cuda, reference):
    curves = np.stack([prep(reference, FAM[k], 64, k + 1) for k in range(4)])
    d = cva.elastic_distance_matrix(curves)
    i, j = np.meshgrid(np.arange(4), np.arange(4), indexing="ij")
    g = cva.elastic_approach2_batch(curves[i.ravel()], curves[j.ravel()])
    np.testing.assert_array_equal(d.ravel(), g["distance"])


def test_elastic_errors(cuda, reference):  # test_elastic.cpp:103-111
    a = prep(reference, "circle", 64)
    with pytest.raises(ValueError):
        cva.elastic_distance_approach2(a, a[:32])
    tiny = a[:4]
    with pytest.raises(ValueError):
        cva.elastic_distance_approach2(tiny, tiny)
    with pytest.raises(ValueError):
        cva.distance_matrix([a], 64)
    bad = a.copy()
    bad[3, 0] = np.nan
    r = cva.elastic_approach2_batch(np.stack([a, bad]), np.stack([a, a]))
    assert r["status"][0] == 0 and r["status"][1] != 0 and np.isnan(r["distance"][1])


def test_golden_fixtures(cuda):
    """The committed reference outputs (tests/golden/elastic_kat.npz) on the GPU:
    DP bitwise, approach 2 and distance_matrix within the rule above."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "elastic_kat.npz"))
    for n in (16, 48):
        gam, e, st = cva.dp_reparam_batch(g[f"dp{n}_q1"], g[f"dp{n}_q2"])
        np.testing.assert_array_equal(gam, g[f"dp{n}_gamma"])
        np.testing.assert_array_equal(e, g[f"dp{n}_energy"])
    r = cva.elastic_approach2_batch(g["a2_c1"], g["a2_c2"], return_gamma=True)
    np.testing.assert_allclose(r["distance"], g["a2_distance"], rtol=DIST_RTOL, atol=1e-12)
    np.testing.assert_array_equal(r["iterations"], g["a2_iterations"])
    d = cva.distance_matrix(list(g["dm_raw"]), 64)
    np.testing.assert_allclose(d, g["dm_d"], rtol=DIST_RTOL, atol=1e-12)


# ---------------------------------------------------------------- approach 1


@pytest.mark.parametrize("n", [32, 48, 64])
def test_approach1_matches_reference(cuda, reference, n):
    c1, c2 = _pairs(reference, n, 5, seed0=41)
    g = cva.elastic_approach1_batch(c1, c2, return_gamma=True)
    r = reference.elastic_approach1_batch(c1, c2, threads=8, gamma=True)
    assert (g["status"] == 0).all() and (r["status"] == 0).all()
    np.testing.assert_allclose(g["distance"], r["distance"], rtol=DIST_RTOL, atol=1e-12)
    # same winning start shift, unless two shifts tie to rounding (symmetric
    # shapes: hippopede / limacon pairs tie at m and m + n/2); the distances
    # agree either way (asserted above)
    same = g["t0"] == r["t0"]
    assert same.sum() >= len(same) - 1
    np.testing.assert_allclose(g["theta"][same], r["theta"][same], atol=1e-12)
    assert (g["iterations"] == 1).all() and (g["converged"] == 1).all()


def test_approach1_golden_and_limit(cuda):
    import os

    gl = np.load(os.path.join(os.path.dirname(__file__), "golden", "elastic_kat.npz"))
    r = cva.elastic_approach1_batch(gl["a1_c1"], gl["a1_c2"], return_gamma=True)
    np.testing.assert_allclose(r["distance"], gl["a1_distance"], rtol=DIST_RTOL, atol=1e-12)
    with pytest.raises(ValueError):  # elastic.cpp:66-69
        cva.elastic_distance_approach1(gl["a1_c1"][0], gl["a1_c2"][0], n_max_approach1=16)


def test_distance_matrix_approach1_matches_reference(cuda, reference):
    raw = np.stack([reference.gen_curve(FAM[k], 200, seed=k + 1) for k in range(3)])
    d = cva.distance_matrix(list(raw), 32, method=1)
    rd = reference.distance_matrix(raw, 32, method=1, threads=4)
    np.testing.assert_allclose(d, rd, rtol=DIST_RTOL, atol=1e-12)


# ------------------------------------------------------------ SRV utilities


def test_srv_utilities_match_reference(cuda, reference):  # test_srv.cpp:130-176
    q = reference.srv_transform(prep(reference, "bumps", 64, 3))
    q2 = reference.srv_transform(prep(reference, "limacon", 64, 4))
    ident = np.arange(65) / 64
    np.testing.assert_array_equal(cva.apply_srv_action(q, 0.0, 0.0, ident), q)  # identity action
    np.testing.assert_array_equal(cva.apply_srv_action(q, 0.0, 0.0, ident),
                                  reference.apply_srv_action(q, 0.0, 0.0, ident))
    gam, _ = cva.dp_reparam(q, q2)
    a = cva.apply_srv_action(q, 0.37, 1.1, gam)
    b = reference.apply_srv_action(q, 0.37, 1.1, gam)
    assert np.abs(a - b).max() <= 1e-14 * np.abs(b).max()  # CUDA cos/sin vs glibc: ulps
    e_g = cva.elastic_energy(q, q2, 0.37, 1.1, gam)
    assert e_g == pytest.approx(reference.elastic_energy(q, q2, 0.37, 1.1, gam), rel=1e-13)
    for (i0, j0, di, dj) in [(0, 0, 1, 1), (5, 7, 3, 2), (60, 63, 4, 3), (130, 3, 2, 3)]:
        assert cva.dp_step_cost(q, q2, i0, j0, di, dj) == reference.dp_step_cost(q, q2, i0, j0, di, dj)
    with pytest.raises(ValueError):
        cva.dp_step_cost(q, q2, 0, 0, 0, 1)
    with pytest.raises(ValueError):
        cva.apply_srv_action(q, 0.0, 0.0, ident[::-1])  # not a monotone warp (srv.cpp:58-69)


# ------------------------------------------------- other shapes of the kernels


def test_dp_n512_global_parent_slab(cuda, reference):
    """n = 512: the DP parents no longer fit in shared memory and go to a
    per-CTA global slab; still bitwise the reference."""
    q1, q2 = srv_pair(reference, 512, 3)
    g, e, st = cva.dp_reparam_batch(q1[None], q2[None])
    rg, re_, rst = reference.dp_reparam_batch(q1[None], q2[None])
    assert st[0] == rst[0] == 0
    np.testing.assert_array_equal(g, rg)
    np.testing.assert_array_equal(e, re_)


def test_approach2_n512_matches_reference(cuda, reference):
    c1, c2 = _pairs(reference, 512, 2, seed0=61)
    _check_vs_reference(cva.elastic_approach2_batch(c1, c2), reference.elastic_approach2_batch(c1, c2, threads=2))


@pytest.mark.parametrize("w", [2, 3])
def test_approach2_other_slopes_match_reference(cuda, reference, w):
    c1, c2 = _pairs(reference, 64, 4, seed0=71)
    g = cva.elastic_approach2_batch(c1, c2, max_slope=w)
    r = reference.elastic_approach2_batch(c1, c2, max_slope=w, threads=4)
    _check_vs_reference(g, r)


def test_approach2_iteration_cap_and_tolerance(cuda, reference):
    c1, c2 = _pairs(reference, 64, 4, seed0=81)
    for it, tol in ((1, 1e-6), (3, 0.0), (0, 1e-6)):
        g = cva.elastic_approach2_batch(c1, c2, max_iters=it, energy_tol=tol)
        r = reference.elastic_approach2_batch(c1, c2, max_iters=it, energy_tol=tol, threads=4)
        _check_vs_reference(g, r)


# ------------------------------------------- slab mode (n or W past shared memory)
# Every per-pair array, the dp ring and the parents in a per-CTA global slab;
# the rigid steps by the direct correlation (elastic.cu align_direct).


@pytest.mark.parametrize("n", [1025, 1100, 2048])
def test_dp_slab_mode_bitwise(cuda, reference, n):
    q1, q2 = srv_pair(reference, n, 5)
    g, e, st = cva.dp_reparam_batch(q1[None], q2[None])
    rg, re_, rst = reference.dp_reparam_batch(q1[None], q2[None])
    assert st[0] == rst[0] == 0
    np.testing.assert_array_equal(g, rg)
    np.testing.assert_array_equal(e, re_)


@pytest.mark.parametrize("w", [9, 12, 20])
def test_dp_large_slopes_bitwise(cuda, reference, w):
    pairs = [srv_pair(reference, 48, s) for s in (2, 3)]
    q1 = np.stack([p[0] for p in pairs])
    q2 = np.stack([p[1] for p in pairs])
    g, e, st = cva.dp_reparam_batch(q1, q2, max_slope=w)
    rg, re_, rst = reference.dp_reparam_batch(q1, q2, max_slope=w)
    assert (st == 0).all() and (rst == 0).all()
    np.testing.assert_array_equal(g, rg)
    np.testing.assert_array_equal(e, re_)


def test_dp_slope_beyond_parent_range_unsupported(cuda, reference):
    q1, q2 = srv_pair(reference, 48, 2)
    with pytest.raises(Exception, match="max_slope"):
        cva.dp_reparam_batch(q1[None], q2[None], max_slope=21)


@pytest.mark.parametrize("n", [1100, 1536])
def test_approach2_slab_mode_matches_reference(cuda, reference, n):
    c1, c2 = _pairs(reference, n, 2, seed0=91)
    g = cva.elastic_approach2_batch(c1, c2, max_iters=4, return_gamma=True)
    r = reference.elastic_approach2_batch(c1, c2, max_iters=4, threads=2, gamma=True)
    _check_vs_reference(g, r)
    np.testing.assert_allclose(g["t0"], r["t0"], atol=1e-9)
    assert (g["gamma"][:, 0] == 0).all() and (g["gamma"][:, -1] == 1).all()


def test_approach2_slab_mode_small_n_agrees_with_shared_kernel(cuda, reference):
    """W = 9 forces slab mode at n = 64 (direct correlation, global step
    table); the same pairs at W = 9 against the reference, and W = 4 slab vs
    shared cannot be compared (different W), so the check is the reference."""
    c1, c2 = _pairs(reference, 64, 4, seed0=101)
    g = cva.elastic_approach2_batch(c1, c2, max_slope=9)
    r = reference.elastic_approach2_batch(c1, c2, max_slope=9, threads=4)
    _check_vs_reference(g, r)


def test_distance_matrix_slab_mode(cuda, reference):
    curves = np.stack([prep(reference, f, 1030, s) for s, f in enumerate(["bumps", "clover", "limacon"], 1)])
    d = cva.elastic_distance_matrix(curves, 2, max_iters=3)
    i, j = np.meshgrid(np.arange(3), np.arange(3), indexing="ij")
    r = reference.elastic_approach2_batch(curves[i.ravel()], curves[j.ravel()], max_iters=3, threads=9)
    np.testing.assert_allclose(d.ravel(), r["distance"], rtol=DIST_RTOL, atol=1e-12)


def test_approach1_slab_mode_matches_reference(cuda, reference):
    c1, c2 = _pairs(reference, 40, 2, seed0=111)
    g = cva.elastic_approach1_batch(c1, c2, max_slope=9)
    r = reference.elastic_approach1_batch(c1, c2, max_slope=9, threads=2)
    assert (g["status"] == 0).all() and (r["status"] == 0).all()
    np.testing.assert_allclose(g["distance"], r["distance"], rtol=DIST_RTOL, atol=1e-12)
    np.testing.assert_array_equal(g["t0"], r["t0"])


@pytest.mark.parametrize("n", [64, 100, 256])
def test_approach2_naive_correlation_matches_reference(cuda, reference, n):
    """ElasticOptions::use_fft = false: the rigid steps run on the direct
    per-shift sums (align_naive, rigid_align.cpp:198-202), on both sides."""
    c1, c2 = _pairs(reference, n, 4, seed0=121)
    g = cva.elastic_approach2_batch(c1, c2, use_fft=False)
    r = reference.elastic_approach2_batch(c1, c2, use_fft=False, threads=4)
    _check_vs_reference(g, r)


def test_distance_matrix_naive_correlation(cuda, reference):
    curves = np.stack([prep(reference, f, 64, s) for s, f in enumerate(["bumps", "clover", "limacon"], 1)])
    d = cva.elastic_distance_matrix(curves, 2, use_fft=False)
    i, j = np.meshgrid(np.arange(3), np.arange(3), indexing="ij")
    r = reference.elastic_approach2_batch(curves[i.ravel()], curves[j.ravel()], use_fft=False, threads=9)
    np.testing.assert_allclose(d.ravel(), r["distance"], rtol=DIST_RTOL, atol=1e-12)
