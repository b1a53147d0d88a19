"""CPU: the C restatement of the elastic rows (oracle/elastic_oracle.c) pinned
bitwise to the reference's own code — against the committed golden vectors
(tests/golden/elastic_kat.npz, made by tools/make_golden.py from oracle/_ref)
and, where oracle/_ref is built, live."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "elastic_kat.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


@pytest.mark.parametrize("n", [16, 48])
def test_dp_golden_bitwise(oracle, g, n):  # acceptance.cpp:296-330, :483-497
    gam, e, st = oracle.dp_reparam_batch(g[f"dp{n}_q1"], g[f"dp{n}_q2"])
    assert (st == 0).all()
    np.testing.assert_array_equal(gam, g[f"dp{n}_gamma"])
    np.testing.assert_array_equal(e, g[f"dp{n}_energy"])


@pytest.mark.parametrize("w", [1, 2, 3, 5])
def test_dp_slopes_golden_bitwise(oracle, g, w):
    gam, e, st = oracle.dp_reparam_batch(g["dp48_q1"][:1], g["dp48_q2"][:1], max_slope=w)
    np.testing.assert_array_equal(gam[0], g[f"dp48_w{w}_gamma"])
    assert e[0] == g[f"dp48_w{w}_energy"]


def test_dp_is_the_exhaustive_minimum(oracle, g):  # acceptance.cpp:296-330 (criterion 8)
    """The DP energy equals the minimum over all admissible lattice paths,
    enumerated with the same per-step costs (n = 16)."""
    q1, q2 = g["dp16_q1"][0], g["dp16_q2"][0]
    n, W = 16, 4
    steps = [(a, b) for a in range(1, W + 1) for b in range(1, W + 1) if np.gcd(a, b) == 1]
    best = {(0, 0): 0.0}
    for i in range(1, n + 1):
        for j in range(1, n + 1):
            cands = [best[(i - a, j - b)] + oracle.dp_step_cost(q1, q2, i - a, j - b, a, b)
                     for a, b in steps if (i - a, j - b) in best]
            if cands:
                best[(i, j)] = min(cands)
    assert best[(n, n)] == g["dp16_energy"][0]


def test_action_and_energy_golden_bitwise(oracle, g):  # test_srv.cpp:130-170
    np.testing.assert_array_equal(oracle.apply_srv_action(g["act_q"], 0.37, 1.1, g["act_gamma"]), g["act_out"])
    ident = oracle.apply_srv_action(g["act_q"], 0.0, 0.0, np.arange(65) / 64)
    np.testing.assert_array_equal(ident, g["act_out_identity"])
    np.testing.assert_array_equal(ident, g["act_q"])  # identity action returns the samples (test_srv.cpp:130-137)
    e = oracle.elastic_energy(g["act_q"], g["act_q2"], 0.37, 1.1, g["act_gamma"])
    assert e == g["act_energy"][0]


def test_approach2_golden_bitwise(oracle, g):  # elastic.cpp:102-174
    r = oracle.elastic_approach2_batch(g["a2_c1"], g["a2_c2"], gamma=True)
    for k in ("distance", "energy", "t0", "theta", "iterations", "converged", "gamma"):
        np.testing.assert_array_equal(r[k], g[f"a2_{k}"], err_msg=k)


def test_approach2_properties(oracle, g):  # acceptance.cpp:455-470
    r = oracle.elastic_approach2_batch(g["a2_c1"], g["a2_c2"], gamma=True)
    assert (r["distance"] >= 0).all() and np.allclose(r["distance"], np.sqrt(r["energy"]), rtol=1e-15)
    assert (np.diff(r["gamma"], axis=1) >= 0).all()
    c = g["a2_c1"][0]
    same = oracle.elastic_approach2_batch(c[None], c[None])
    assert same["distance"][0] < 1e-6  # test_elastic.cpp:35-40


def test_oracle_elastic_matches_reference_live(oracle, reference, g):
    c1, c2 = g["a2_c1"][:3], g["a2_c2"][:3]
    r, o = reference.elastic_approach2_batch(c1, c2), oracle.elastic_approach2_batch(c1, c2)
    np.testing.assert_array_equal(r["distance"], o["distance"])
    q1, q2 = g["dp48_q1"], g["dp48_q2"]
    np.testing.assert_array_equal(reference.dp_reparam_batch(q1, q2)[0], oracle.dp_reparam_batch(q1, q2)[0])


def test_approach1_golden_bitwise(oracle, g):  # elastic.cpp:62-100
    r = oracle.elastic_approach1_batch(g["a1_c1"], g["a1_c2"], gamma=True)
    for k in ("distance", "energy", "t0", "theta", "gamma"):
        np.testing.assert_array_equal(r[k], g[f"a1_{k}"], err_msg=k)
    assert (r["iterations"] == 1).all() and (r["converged"] == 1).all()


def test_approach1_limit(oracle, g):  # elastic.cpp:66-69
    r = oracle.elastic_approach1_batch(g["a1_c1"][:1], g["a1_c2"][:1], n_max=16)
    assert r["status"][0] == 1
