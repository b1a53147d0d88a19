"""CPU: pin the oracle (oracle/curvalign_oracle.c) against the reference.

Two independent pins:
* the committed golden vectors (tests/golden/, produced by the reference's own
  code via tools/make_golden.py), checked here without the reference present;
* the reference compiled in place (oracle/_ref), run live on seeded inputs.
The known-answer tests restate the reference's own unit tests (file:line cited).
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PI = np.pi


def gold(name):
    return np.load(os.path.join(GOLD, name))


def wrap(a):
    return (a + PI) % (2 * PI) - PI


def assert_res_equal(r, g, tol=1e-12):
    assert int(r["shift"]) == int(g["shift"])
    assert abs(wrap(float(r["theta"]) - float(g["theta"]))) <= tol
    assert abs(float(r["trace"]) - float(g["trace"])) <= tol * max(1.0, abs(float(g["trace"])))
    assert abs(float(r["energy"]) - float(g["energy"])) <= tol * max(1.0, abs(float(g["energy"])))


# ---------------------------------------------------------------- rigid_align


def test_diamond_correlation(oracle):  # test_rigid_align.cpp:47-56
    g = gold("rigid_align_kat.npz")
    a = oracle.cross_correlation_matrix(g["diamond"], g["diamond"], 1)
    np.testing.assert_allclose(a, [0.0, 2.0, -2.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(a, g["diamond_A1"], atol=1e-15)


def test_closed_form_known_matrix(oracle):  # test_rigid_align.cpp:79-86
    th, tr, dg = oracle.optimal_rotation([0.0, 1.0, -1.0, 0.0], svd=False)
    assert th == pytest.approx(PI / 2, abs=1e-14) and tr == pytest.approx(2.0) and not dg
    th2, tr2, dg2 = oracle.optimal_rotation([0.0, 1.0, -1.0, 0.0], svd=True)
    assert th2 == pytest.approx(PI / 2, abs=1e-14) and tr2 == pytest.approx(2.0) and not dg2


def test_svd_matches_closed_form(oracle):  # test_rigid_align.cpp:88-100
    rng = np.random.default_rng(23)
    for _ in range(1000):
        a = rng.uniform(-2, 2, 4)
        th_s, tr_s, _ = oracle.optimal_rotation(a, svd=True)
        th_c, tr_c, _ = oracle.optimal_rotation(a, svd=False)
        assert abs(tr_s - tr_c) < 1e-10
        if abs(tr_s) > 1e-6:
            assert abs(wrap(th_s - th_c)) < 1e-8


def test_degenerate_flagged(oracle):  # test_rigid_align.cpp:102-108
    assert oracle.optimal_rotation([0, 0, 0, 0], svd=True)[2]
    assert oracle.optimal_rotation([0, 0, 0, 0], svd=False)[2]


@pytest.mark.parametrize("case", ["limacon", "fourier", "bumps"])
def test_recovery_fixtures(oracle, case):  # test_rigid_align.cpp:153-185, test_synthetic.cpp:100-107
    g = gold("rigid_align_kat.npz")
    r = oracle.align(g[f"{case}_c1"], g[f"{case}_c2"])
    assert_res_equal(r, g[f"{case}_res"][0])
    if case == "limacon":
        assert r["shift"] == 29 and abs(r["theta"]) < 1e-9 and r["energy"] < 1e-15
    else:
        assert r["t0"] == pytest.approx(0.25, abs=1e-12)
        assert r["theta"] == pytest.approx(PI / 3, abs=1e-9)


def test_circle_tie_break(oracle):  # test_rigid_align.cpp:170-176
    g = gold("rigid_align_kat.npz")
    r = oracle.align(g["circle"], g["circle"])
    assert r["shift"] == 0 and abs(r["theta"]) < 1e-9 and r["energy"] < 1e-12
    assert_res_equal(r, g["circle_res"][0])


def test_rotation_covariance(oracle):  # test_rigid_align.cpp:212-220
    g = gold("rigid_align_kat.npz")
    base = oracle.align(g["hippo_c1"], g["hippo_c1"])
    rot = oracle.align(g["hippo_c1"], g["hippo_c2"])
    assert rot["shift"] == base["shift"]
    assert wrap(rot["theta"] - base["theta"]) == pytest.approx(0.4, abs=1e-8)
    assert_res_equal(rot, g["hippo_rot"][0])


def test_reflection_not_undone(oracle):  # test_rigid_align.cpp:237-246
    g = gold("rigid_align_kat.npz")
    r = oracle.align(g["reflect_c1"], g["reflect_c2"])
    assert r["energy"] > 1e-6
    assert_res_equal(r, g["reflect_res"][0])


@pytest.mark.parametrize("n", [8, 20, 64, 101, 128, 1024])
def test_naive_equals_fft(oracle, n):  # test_rigid_align.cpp:133-151
    g = gold("rigid_align_kat.npz")
    a, b = g[f"rand{n}_c1"], g[f"rand{n}_c2"]
    naive = oracle.correlation_all_shifts(a, b, fft=False)
    fft = oracle.correlation_all_shifts(a, b, fft=True)
    assert np.abs(naive - fft).max() < 1e-9 * n
    np.testing.assert_allclose(naive, g[f"rand{n}_naive"], atol=1e-12)
    np.testing.assert_allclose(fft, g[f"rand{n}_fft"], atol=1e-12)
    assert_res_equal(oracle.align(a, b), g[f"rand{n}_res"][0])
    assert_res_equal(oracle.align(a, b, fft=False), g[f"rand{n}_res_naive"][0])


def test_energy_identity_matches_direct(oracle):  # test_rigid_align.cpp:187-197
    rng = np.random.default_rng(57)
    a, b = rng.uniform(-1, 1, (48, 2)), rng.uniform(-1, 1, (48, 2))
    r = oracle.align(a, b, fft=False)
    direct = oracle.mismatch_energy(a, b, int(r["shift"]), float(r["theta"]))
    assert r["energy"] == pytest.approx(direct, rel=1e-9)


def test_input_validation(oracle):  # test_rigid_align.cpp:248-257
    c32, c64 = np.zeros((32, 2)), np.zeros((64, 2))
    with pytest.raises(ValueError):
        oracle.align(c32, c64)
    with pytest.raises(ValueError):
        oracle.cross_correlation_matrix(c32, c32, 32)
    with pytest.raises(ValueError):
        oracle.align(np.array([[0, 0], [1, 0], [0, 1.0]]), np.array([[0, 0], [1, 0], [0, 1.0]]))


def test_fft_matches_numpy(oracle):
    rng = np.random.default_rng(5)
    for n in (2, 3, 8, 20, 33, 101, 1024, 4097):
        x = rng.standard_normal(n)
        np.testing.assert_allclose(oracle.real_dft(x), np.fft.rfft(x), atol=1e-12 * n)
        y = rng.standard_normal(n)
        want = np.real(np.fft.ifft(np.conj(np.fft.fft(x)) * np.fft.fft(y)))
        np.testing.assert_allclose(oracle.circular_cross_correlation(x, y), want, atol=1e-12 * n)


# ------------------------------------------------------------------ curve core


def test_arc_length_known(oracle):  # test_curve_core.cpp:126-138
    g = gold("curve_core_kat.npz")
    s, tot = oracle.arc_length_params(g["square"])
    np.testing.assert_allclose(s, [0, 0.25, 0.5, 0.75, 1.0], atol=1e-15)
    assert tot == pytest.approx(4.0)
    s, _ = oracle.arc_length_params(g["rect"])
    np.testing.assert_allclose(s, [0, 1 / 3, 0.5, 5 / 6, 1.0], atol=1e-15)
    s, _ = oracle.arc_length_params(g["clover200"])
    np.testing.assert_array_equal(s, g["clover200_s"])
    assert np.all(np.diff(s) > 0) and s[0] == 0.0 and s[-1] == 1.0


def test_coincident_nodes_rejected(oracle):  # test_curve_core.cpp:140-144
    with pytest.raises(ValueError):
        oracle.arc_length_params(np.array([[0, 0], [1, 0], [1, 0], [0, 1.0]]))


def test_spline_golden(oracle):  # test_curve_core.cpp:36-44
    g = gold("curve_core_kat.npz")
    v = oracle.spline(g["spline_x"], g["spline_y"], g["spline_xq"])
    np.testing.assert_allclose(v, g["spline_val"], rtol=0, atol=1e-14)
    knots = oracle.spline(g["spline_x"], g["spline_y"], g["spline_x"][:-1])
    np.testing.assert_allclose(knots, g["spline_y"][:-1], atol=1e-14)


@pytest.mark.parametrize("name,n_out", [("nonuniform_circle", 256), ("gon128", 128)])
def test_resample_golden(oracle, name, n_out):  # test_curve_core.cpp:154-189
    g = gold("curve_core_kat.npz")
    r = oracle.resample_uniform(g[name], n_out)
    np.testing.assert_allclose(r, g[f"{name}_r{n_out}"], atol=1e-14)


def test_preprocess_golden(oracle):  # test_curve_core.cpp:215-232
    g = gold("curve_core_kat.npz")
    np.testing.assert_allclose(oracle.preprocess(g["hippo100"], 128), g["hippo100_prep128"], atol=1e-15)
    np.testing.assert_allclose(oracle.preprocess(g["hippo100"], 64, resample=False),
                               g["hippo100_prep_noresample"], atol=1e-15)
    np.testing.assert_allclose(oracle.preprocess(g["square"], 8), g["square_prep8"], atol=1e-15)


def test_srv_golden(oracle):  # test_srv.cpp:80-128
    g = gold("srv_kat.npz")
    q = oracle.srv_transform(g["circle_prep256"])
    np.testing.assert_allclose(q, g["circle_q"], atol=1e-14)
    assert np.all(np.abs(np.hypot(q[:, 0], q[:, 1]) - 1.0) < 1e-3)
    qc = oracle.srv_center(oracle.srv_transform(g["bumps_prep128"]))
    np.testing.assert_allclose(qc, g["bumps_qc"], atol=1e-14)
    assert np.hypot(*qc.mean(0)) < 1e-12


# ------------------------------------------------------------ config samples


def test_config_samples_golden(oracle):
    g = gold("configs_sample.npz")
    # C0: preprocess(resample=false) + align
    pts = np.concatenate([g["c0_c1"], g["c0_c2"]])
    res, al = oracle.batch(pts, [0, 256, 512], 256, mode=0, resample=False, aligned=True)
    assert_res_equal(res[0], g["c0_res"][0])
    np.testing.assert_allclose(al, g["c0_aligned"], atol=1e-13)
    # C1 sample
    res, al = oracle.batch(g["c1_points"], g["c1_offsets"], 1024, mode=0, aligned=True)
    for r, gg in zip(res, g["c1_res"]):
        assert_res_equal(r, gg)
    np.testing.assert_allclose(al, g["c1_aligned"], atol=1e-13)
    # C2 sample
    prep = np.stack([oracle.preprocess(g["c2_points"][g["c2_offsets"][i]:g["c2_offsets"][i + 1]], 512)
                     for i in range(6)])
    np.testing.assert_allclose(prep, g["c2_prep"], atol=1e-15)
    for i in range(6):
        for j in range(6):
            r = oracle.align(prep[i], prep[j])
            assert int(r["shift"]) == int(g["c2_shift"][i, j])
            assert r["energy"] == pytest.approx(g["c2_energy"][i, j], rel=1e-12, abs=1e-15)
    # C4 sample
    pts = np.concatenate([g["c4_c1"][0], g["c4_c2"][0], g["c4_c1"][1], g["c4_c2"][1]])
    res, al = oracle.batch(pts, [0, 2048, 4096, 6144, 8192], 2048, mode=2, aligned=True)
    for r, gg in zip(res, g["c4_res"]):
        assert_res_equal(r, gg)
    np.testing.assert_allclose(al, g["c4_aligned"], atol=1e-13)


# ------------------------------------------------------- live reference pins


def test_oracle_matches_reference_live(oracle, reference):
    from paper_2501_17779_b200 import synth

    pts, offs, _, _ = synth.ragged_pairs(123, 24, 1024)
    ro, ao = oracle.batch(pts, offs, 1024, mode=0, threads=4, aligned=True)
    rr, ar = reference.batch(pts, offs, 1024, mode=0, threads=4, aligned=True)
    np.testing.assert_array_equal(ro["shift"], rr["shift"])
    np.testing.assert_allclose(ro["theta"], rr["theta"], atol=1e-13)
    np.testing.assert_allclose(ro["energy"], rr["energy"], atol=1e-16, rtol=1e-12)
    np.testing.assert_allclose(ao, ar, atol=1e-13)
    rng = np.random.default_rng(9)
    for n in (4, 5, 9, 37, 100, 255, 256):
        a, b = rng.uniform(-1, 1, (n, 2)), rng.uniform(-1, 1, (n, 2))
        assert_res_equal(oracle.align(a, b), reference.align(a, b))
        if n >= 8:
            walk = np.cumsum(a, 0)
            np.testing.assert_allclose(oracle.srv_transform(walk), reference.srv_transform(walk), atol=1e-12)
