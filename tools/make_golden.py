"""Generate tests/golden/*.npz from the REFERENCE's own code (oracle/_ref).

Run here (where /root/reference exists and `make ref` built oracle/_ref):
    python tools/make_golden.py
Each fixture holds inputs plus the reference's outputs for them; the oracle
(tests/test_oracle_pins.py) and the GPU path (tests/test_gpu_*.py) are checked
against these files. Cases restate the reference's own known-answer tests
(proj/tests/test_rigid_align.cpp, test_curve_core.cpp, test_srv.cpp,
test_synthetic.cpp) plus small seeded samples of the BASELINE configs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from pyoracle import ALIGNMENT_DTYPE, Reference  # noqa: E402

from paper_2501_17779_b200 import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
PI = np.pi


def rec(a):
    return np.array([tuple(a)], dtype=ALIGNMENT_DTYPE)


def aligned_of(c2, r):
    n = c2.shape[0]
    c, s = np.cos(r["theta"]), np.sin(r["theta"])
    q = c2[(np.arange(n) + int(r["shift"])) % n]
    return np.stack([c * q[:, 0] + s * q[:, 1], -s * q[:, 0] + c * q[:, 1]], 1)


def main():
    R = Reference()
    os.makedirs(OUT, exist_ok=True)
    kat = {}

    # --- rigid_align known answers (proj/tests/test_rigid_align.cpp)
    diamond = np.array([[1, 0], [0, 1], [-1, 0], [0, -1]], float)
    kat["diamond"] = diamond
    kat["diamond_A1"] = R.cross_correlation_matrix(diamond, diamond, 1)  # :47-56

    lim = R.gen_curve("limacon", 96)  # :153-168
    lim2 = np.empty_like(lim)
    for l in range(96):
        lim2[(l + 29) % 96] = lim[l]
    kat["limacon_c1"], kat["limacon_c2"] = lim, lim2
    kat["limacon_res"] = rec(R.align(lim, lim2))

    circ = R.gen_curve("circle", 64)  # :170-176
    kat["circle"] = circ
    kat["circle_res"] = rec(R.align(circ, circ))

    f1 = R.gen_curve("fourier_random", 256, 5)  # :178-185
    f2 = R.transform_curve(f1, 0.25, PI / 3.0)
    kat["fourier_c1"], kat["fourier_c2"] = f1, f2
    kat["fourier_res"] = rec(R.align(f1, f2))

    b1 = R.gen_curve("bumps", 256)  # test_synthetic.cpp:100-107
    b2 = R.transform_curve(b1, 0.25, PI / 3.0)
    kat["bumps_c1"], kat["bumps_c2"] = b1, b2
    kat["bumps_res"] = rec(R.align(b1, b2))

    h1 = R.gen_curve("hippopede", 128)  # :212-220
    h2 = h1.copy()
    c, s = np.cos(0.4), np.sin(0.4)
    h2 = np.stack([c * h1[:, 0] - s * h1[:, 1], s * h1[:, 0] + c * h1[:, 1]], 1)
    kat["hippo_c1"], kat["hippo_c2"] = h1, h2
    kat["hippo_base"] = rec(R.align(h1, h1))
    kat["hippo_rot"] = rec(R.align(h1, h2))

    lr = R.gen_curve("limacon", 128)  # :237-246
    lm = lr.copy()
    lm[:, 1] = -lm[:, 1]
    kat["reflect_c1"], kat["reflect_c2"] = lr, lm
    kat["reflect_res"] = rec(R.align(lr, lm))

    rng = np.random.default_rng(43)  # :133-151 (naive == fft); pow2 and non-pow2 n
    for n in (8, 20, 64, 101, 128, 1024):
        a = rng.uniform(-1, 1, (n, 2))
        b = rng.uniform(-1, 1, (n, 2))
        kat[f"rand{n}_c1"], kat[f"rand{n}_c2"] = a, b
        kat[f"rand{n}_naive"] = R.correlation_all_shifts(a, b, fft=False)
        kat[f"rand{n}_fft"] = R.correlation_all_shifts(a, b, fft=True)
        kat[f"rand{n}_res"] = rec(R.align(a, b))
        kat[f"rand{n}_res_naive"] = rec(R.align(a, b, fft=False))
    np.savez_compressed(os.path.join(OUT, "rigid_align_kat.npz"), **kat)

    # --- curve core / spline known answers (proj/tests/test_curve_core.cpp)
    cc = {}
    sq = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float)
    rect = np.array([[0, 0], [2, 0], [2, 1], [0, 1]], float)
    cc["square"], cc["rect"] = sq, rect
    cc["square_s"], cc["square_len"] = R.arc_length_params(sq)
    cc["rect_s"], cc["rect_len"] = R.arc_length_params(rect)
    cc["square_resampled8"] = R.resample_uniform(sq, 8)
    cc["square_prep8"] = R.preprocess(sq, 8)
    x = np.array([0.0, 0.2, 0.45, 0.7, 1.0])
    y = np.array([1.0, -0.5, 2.0, 0.25, 1.0])
    xq = np.linspace(-0.3, 1.3, 41)
    cc["spline_x"], cc["spline_y"], cc["spline_xq"] = x, y, xq
    cc["spline_val"] = R.spline(x, y, xq)
    nonu = np.array([[np.cos(2 * PI * (t + 0.15 * t * (1 - t))), np.sin(2 * PI * (t + 0.15 * t * (1 - t)))]
                     for t in np.arange(64) / 64.0])
    cc["nonuniform_circle"] = nonu
    cc["nonuniform_circle_r256"] = R.resample_uniform(nonu, 256)
    gon = np.array([[np.cos(2 * PI * i / 128), np.sin(2 * PI * i / 128)] for i in range(128)])
    cc["gon128"] = gon
    cc["gon128_r128"] = R.resample_uniform(gon, 128)
    hip = R.gen_curve("hippopede", 100)
    cc["hippo100"] = hip
    cc["hippo100_prep128"] = R.preprocess(hip, 128)
    cc["hippo100_prep_noresample"] = R.preprocess(hip, 64, resample=False)
    clover = R.gen_curve("clover", 200)
    cc["clover200"] = clover
    cc["clover200_s"], _ = R.arc_length_params(clover)
    np.savez_compressed(os.path.join(OUT, "curve_core_kat.npz"), **cc)

    # --- srv (proj/tests/test_srv.cpp:80-128)
    sv = {}
    circ_p = R.preprocess(R.gen_curve("circle", 512), 256)
    sv["circle_prep256"] = circ_p
    sv["circle_q"] = R.srv_transform(circ_p)
    bp = R.preprocess(R.gen_curve("bumps", 256), 128)
    sv["bumps_prep128"] = bp
    sv["bumps_qc"] = R.srv_center(R.srv_transform(bp))
    np.savez_compressed(os.path.join(OUT, "srv_kat.npz"), **sv)

    # --- BASELINE config samples (seeded synthetic inputs, reference outputs)
    cfg = {}
    c1, c2, k, th = synth.uniform_pairs(7, 1, 256, modes=7, sigma=1e-3)  # C0
    pts = np.concatenate([c1[0], c2[0]])
    offs = np.array([0, 256, 512], np.int64)
    res, al = R.batch(pts, offs, 256, mode=0, resample=False, aligned=True)
    cfg["c0_c1"], cfg["c0_c2"], cfg["c0_k"], cfg["c0_theta"] = c1[0], c2[0], k, th
    cfg["c0_res"], cfg["c0_aligned"] = res, al
    pts, offs, k, th = synth.ragged_pairs(11, 4, 1024)  # C1 sample
    res, al = R.batch(pts, offs, 1024, mode=0, resample=True, aligned=True)
    cfg["c1_points"], cfg["c1_offsets"], cfg["c1_k"], cfg["c1_theta"] = pts, offs, k, th
    cfg["c1_res"], cfg["c1_aligned"] = res, al
    cpts, coffs = synth.ragged_curves(13, 6)  # C2 sample: 6 curves -> 36 ordered pairs at N=512
    prep = np.stack([R.preprocess(cpts[coffs[i]:coffs[i + 1]], 512) for i in range(6)])
    e, kk, tt = R.allpairs(prep, 0, 6)
    cfg["c2_points"], cfg["c2_offsets"], cfg["c2_prep"] = cpts, coffs, prep
    cfg["c2_energy"], cfg["c2_shift"], cfg["c2_theta"] = e, kk, tt
    s1, s2, k, th, u = synth.srv_pairs(17, 2, 2048)  # C4 sample
    pts = np.concatenate([s1[0], s2[0], s1[1], s2[1]])
    offs = np.array([0, 2048, 4096, 6144, 8192], np.int64)
    res, al = R.batch(pts, offs, 2048, mode=2, aligned=True)
    cfg["c4_c1"], cfg["c4_c2"], cfg["c4_res"], cfg["c4_aligned"] = s1, s2, res, al
    np.savez_compressed(os.path.join(OUT, "configs_sample.npz"), **cfg)

    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


FAMILIES = ["circle", "superellipse", "hippopede", "bumps", "limacon", "clover", "fourier_random"]


def elastic():
    """tests/golden/elastic_kat.npz: the reference's dp_reparam, apply_srv_action,
    elastic_energy, elastic_distance_approach2 and distance_matrix on seeded
    inputs (restating proj/tests/test_srv.cpp:130-230, test_elastic.cpp:35-150 and
    acceptance.cpp:296-330, :455-530 cases at small sizes)."""
    R = Reference()

    def prep(fam, n, seed):
        return R.preprocess(R.gen_curve(fam, 512, seed=seed), n, True)

    el = {}
    # dp_reparam on SRV pairs (n = 16 as in acceptance.cpp:296-330, 48 as in :483-497)
    for n in (16, 48):
        q1 = np.stack([R.srv_transform(prep("fourier_random", n, s)) for s in range(1, 6)])
        q2 = np.stack([R.srv_transform(prep("fourier_random", n, s + 100)) for s in range(1, 6)])
        g, e, st = R.dp_reparam_batch(q1, q2)
        el[f"dp{n}_q1"], el[f"dp{n}_q2"], el[f"dp{n}_gamma"], el[f"dp{n}_energy"] = q1, q2, g, e
    q1, q2 = el["dp48_q1"][0], el["dp48_q2"][0]
    for w in (1, 2, 3, 5):
        g, e, st = R.dp_reparam_batch(q1[None], q2[None], max_slope=w)
        el[f"dp48_w{w}_gamma"], el[f"dp48_w{w}_energy"] = g[0], e[0]
    # apply_srv_action / elastic_energy with a warp (acceptance.cpp:499-512, test_srv.cpp:150-170)
    q = R.srv_transform(prep("bumps", 64, 3))
    gam = el["dp48_gamma"][0]
    g64 = np.interp(np.arange(65) / 64, np.arange(49) / 48, gam)
    g64[0], g64[-1] = 0.0, 1.0
    el["act_q"], el["act_gamma"] = q, g64
    el["act_out"] = R.apply_srv_action(q, 0.37, 1.1, g64)
    el["act_out_identity"] = R.apply_srv_action(q, 0.0, 0.0, np.arange(65) / 64)
    q2b = R.srv_transform(prep("limacon", 64, 4))
    el["act_q2"], el["act_energy"] = q2b, np.array([R.elastic_energy(q, q2b, 0.37, 1.1, g64)])
    # approach 2 on preprocessed pairs
    c1 = np.stack([prep(FAMILIES[k % 7], 64, k + 1) for k in range(7)])
    c2 = np.stack([prep(FAMILIES[(k + 3) % 7], 64, k + 51) for k in range(7)])
    r = R.elastic_approach2_batch(c1, c2, gamma=True)
    el["a2_c1"], el["a2_c2"] = c1, c2
    for k in ("distance", "energy", "t0", "theta", "iterations", "converged", "gamma"):
        el[f"a2_{k}"] = r[k]
    # approach 1 (exhaustive over start shifts) at n = 32
    a1c1 = np.stack([prep(FAMILIES[k % 7], 32, k + 1) for k in range(5)])
    a1c2 = np.stack([prep(FAMILIES[(k + 3) % 7], 32, k + 51) for k in range(5)])
    r1 = R.elastic_approach1_batch(a1c1, a1c2, gamma=True)
    el["a1_c1"], el["a1_c2"] = a1c1, a1c2
    for k in ("distance", "energy", "t0", "theta", "gamma"):
        el[f"a1_{k}"] = r1[k]
    # distance_matrix(approach2) of 4 raw curves at n = 64 (test_elastic.cpp:113-135)
    raw = np.stack([R.gen_curve(FAMILIES[k], 400, seed=k + 1) for k in range(4)])
    el["dm_raw"], el["dm_d"] = raw, R.distance_matrix_approach2(raw, 64, threads=4)
    np.savez_compressed(os.path.join(OUT, "elastic_kat.npz"), **el)
    print("elastic_kat.npz", os.path.getsize(os.path.join(OUT, "elastic_kat.npz")))


if __name__ == "__main__":
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "elastic":
        elastic()
    else:
        main()
        elastic()
