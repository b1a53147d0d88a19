"""The GPU-vs-reference acceptance rule (BASELINE.json north_star, SURVEY.md
§8(c)) applied to whole batches; shared by tests/test_gpu_full_parity.py and
tools/validate_full.py. Test infrastructure.

  (i)   shift identical, unless the reference's |D| at the two shifts agree
        within 1e-12 relative (a documented near-tie);
  (ii)  |theta_gpu - theta_ref| mod 2 pi <= 1e-10;
  (iii) aligned coordinates: max |a_gpu - a_ref| <= 1e-10 max |a_ref|;
  (iv)  energy: |e_gpu - e_ref| <= 1e-10 e_ref + 1e-14 h (s1 + s2)
        (tests/test_gpu_parity.py explains the absolute term).
"""
import numpy as np

PI = np.pi


def wrap(a):
    return (np.asarray(a) + PI) % (2 * PI) - PI


def tau(c1, c2, m):
    z1 = c1[:, 0] + 1j * c1[:, 1]
    z2 = np.roll(c2[:, 0] + 1j * c2[:, 1], -m)
    return abs(np.sum(np.conj(z1) * z2)) / len(z1)


def compare(res, ro, al, ao, firsts, seconds):
    """res / ro: GPU / reference alignment records; al / ao: aligned curves
    (or None); firsts / seconds: the aligned (preprocessed) inputs. Returns a
    summary dict; `violations` counts pairs outside the rule."""
    n = firsts.shape[1]
    out = {"pairs": int(len(res)), "status_ok": int((res["status"] == 0).sum()), "shift_equal": 0,
           "near_ties": 0, "violations": 0, "max_dtheta": 0.0, "max_coord_rel": 0.0, "max_energy_rel": 0.0}
    out["violations"] += int((res["status"] != 0).sum())
    for p in range(len(res)):
        g, r = res[p], ro[p]
        if int(g["status"]) != 0:
            continue
        c1, c2 = firsts[p], seconds[p]
        if int(g["shift"]) != int(r["shift"]):
            t1, t2 = tau(c1, c2, int(g["shift"])), tau(c1, c2, int(r["shift"]))
            if abs(t1 - t2) <= 1e-12 * max(t1, t2):
                out["near_ties"] += 1
            else:
                out["violations"] += 1
            continue
        out["shift_equal"] += 1
        dth = abs(float(wrap(float(g["theta"]) - float(r["theta"]))))
        out["max_dtheta"] = max(out["max_dtheta"], dth)
        scale = (np.sum(c1 ** 2) + np.sum(c2 ** 2)) / n
        er = abs(float(g["energy"]) - float(r["energy"])) / max(float(r["energy"]), 1e-4 * scale)
        out["max_energy_rel"] = max(out["max_energy_rel"], er)
        cr = 0.0
        if al is not None:
            cr = float(np.abs(al[p] - ao[p]).max() / np.abs(ao[p]).max())
            out["max_coord_rel"] = max(out["max_coord_rel"], cr)
        if dth > 1e-10 or cr > 1e-10 or abs(float(g["energy"]) - float(r["energy"])) > (
                1e-10 * float(r["energy"]) + 1e-14 * scale):
            out["violations"] += 1
    return out


def ragged_of_pairs(a, b):
    """Uniform pairs (a[p], b[p]) as the ragged layout of ref_batch."""
    P, N = a.shape[0], a.shape[1]
    pts = np.empty((P, 2, N, 2))
    pts[:, 0], pts[:, 1] = a, b
    return pts.reshape(-1, 2), np.arange(2 * P + 1, dtype=np.int64) * N
