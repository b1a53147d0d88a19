"""Full-size parity sweep: every pair of the bench's C1 batch (4096 pairs, the
bench's own seed) and of a C4 batch, GPU against the reference's own sources
compiled in place (oracle/_ref), with the acceptance rule of
tests/test_gpu_parity.py applied to every pair. Prints one JSON summary.

    python tools/validate_full.py [--seed 0] [--c4-pairs 2048]

Test infrastructure (reads oracle/ as the checker); not part of the product.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2501_17779_b200 as cva  # noqa: E402
from paper_2501_17779_b200 import synth  # noqa: E402
from pyoracle import Oracle, Reference, reference_available  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests"))
from parity_rule import compare, wrap  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--c4-pairs", type=int, default=2048)
    a = ap.parse_args()
    lib = Reference() if reference_available() else Oracle()
    threads = os.cpu_count() or 1
    summary = {"checker": "reference sources compiled in place" if reference_available() else "C oracle port"}

    cfg = synth.CONFIGS["c1"]
    pts, offs, _, _ = synth.ragged_pairs(a.seed, cfg["pairs"], cfg["N"])
    res, al = cva.preprocess_align_batch(pts, offs, cfg["N"], return_aligned=True)
    ro, ao = lib.batch(pts, offs, cfg["N"], mode=0, threads=threads, aligned=True)
    prep, _ = cva.preprocess_batch(pts, offs, cfg["N"])
    summary["c1"] = compare(res, ro, al, ao, prep[0::2], prep[1::2])

    c1, c2, _, _, _ = synth.srv_pairs(a.seed + 1, a.c4_pairs, 2048)
    res, alq = cva.srv_align_batch(c1, c2, return_aligned=True)
    pts4 = np.concatenate([np.stack([c1[p], c2[p]]) for p in range(a.c4_pairs)]).reshape(-1, 2)
    offs4 = np.arange(2 * a.c4_pairs + 1, dtype=np.int64) * 2048
    ro, ao = lib.batch(pts4, offs4, 2048, mode=2, threads=threads, aligned=True)
    q1 = np.stack([lib.srv_center(lib.srv_transform(c1[p])) for p in range(a.c4_pairs)])
    q2 = np.stack([lib.srv_center(lib.srv_transform(c2[p])) for p in range(a.c4_pairs)])
    summary["c4"] = compare(res, ro, alq, ao, q1, q2)

    # C3: all 256 pairs at N = 65536 (center + normalize, no resampling)
    cfg = synth.CONFIGS["c3"]
    c1, c2, _, _ = synth.uniform_pairs(a.seed + 2, cfg["pairs"], cfg["N"], cfg["modes"], cfg["amp"],
                                       cfg["amp_exp"], cfg["sigma"])
    res, al = cva.preprocess_align_uniform(c1, c2, return_aligned=True)
    pts3 = np.concatenate([np.stack([c1[p], c2[p]]) for p in range(cfg["pairs"])]).reshape(-1, 2)
    offs3 = np.arange(2 * cfg["pairs"] + 1, dtype=np.int64) * cfg["N"]
    ro, ao = lib.batch(pts3, offs3, cfg["N"], mode=0, resample=False, threads=threads, aligned=True)
    u = np.stack([lib.preprocess(c1[p], 0, resample=False) for p in range(cfg["pairs"])])
    v = np.stack([lib.preprocess(c2[p], 0, resample=False) for p in range(cfg["pairs"])])
    summary["c3"] = compare(res, ro, al, ao, u, v)

    # C2: 16 full rows of the 2048 x 2048 matrix (32768 cells) against align_fft
    cfg = synth.CONFIGS["c2"]
    pts2, offs2 = synth.ragged_curves(a.seed + 3, cfg["curves"])
    prep, st = cva.preprocess_batch(pts2, offs2, cfg["N"])
    e, k, th = cva.allpairs(prep)
    rows = np.linspace(0, cfg["curves"] - 1, 16).astype(int)
    M = cfg["curves"]
    a_pts = np.concatenate([np.stack([prep[i], prep[j]]) for i in rows for j in range(M)]).reshape(-1, 2)
    a_offs = np.arange(2 * len(rows) * M + 1, dtype=np.int64) * cfg["N"]
    ro, _ = lib.batch(a_pts, a_offs, cfg["N"], mode=1, resample=False, threads=threads)
    g = np.zeros(len(rows) * M, dtype=ro.dtype)
    g["shift"] = k[rows].ravel()
    g["theta"] = th[rows].ravel()
    g["energy"] = e[rows].ravel()
    g["trace"] = ro["trace"]
    g["t0"] = g["shift"] / cfg["N"]
    firsts = np.repeat(prep[rows], M, axis=0)
    seconds = np.tile(prep, (len(rows), 1, 1))
    dummy = np.ones((len(rows) * M, 1, 2))
    summary["c2_rows"] = compare(g, ro, dummy, dummy, firsts, seconds)

    # E1: every ordered pair of the 64 curves, approach 2 (elastic.cpp:102-174),
    # both sides on the same (reference-preprocessed) curves. Not bitwise (the
    # rigid steps use the FFT correlation): agreement to rounding, same path.
    if reference_available():
        cfg = synth.CONFIGS["e1"]
        M, N = cfg["curves"], cfg["N"]
        pts, offs = synth.ragged_curves(a.seed, M)
        prep = np.stack([lib.preprocess(pts[offs[c]:offs[c + 1]], N, True) for c in range(M)])
        d_gpu = cva.elastic_distance_matrix(prep)
        cells = np.arange(M * M)
        r = lib.elastic_approach2_batch(prep[cells // M], prep[cells % M], threads=threads)
        d_ref = r["distance"].reshape(M, M)
        g2 = cva.elastic_approach2_batch(prep[cells // M], prep[cells % M])
        rel = np.abs(d_gpu - d_ref) / np.maximum(np.abs(d_ref), 1e-300)
        summary["e1"] = {"pairs": int(M * M), "max_distance_rel": float(rel.max()),
                         "median_distance_rel": float(np.median(rel)),
                         "iterations_equal": int((g2["iterations"] == r["iterations"]).sum()),
                         "t0_equal": int((g2["t0"] == r["t0"]).sum()),
                         "max_dtheta": float(np.abs(wrap(g2["theta"] - r["theta"])).max()),
                         "matrix_equals_pair_batch": bool(np.array_equal(d_gpu.ravel(), g2["distance"]))}
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
